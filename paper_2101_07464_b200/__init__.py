"""B200-native Householder Dice (arXiv 2101.07464) hot path.

The product is the CUDA library ``lib/libhd_b200.so`` (sources in ``csrc/``,
C-ABI in ``include/hd.h``). ``paper_2101_07464_b200.lazymat`` mirrors the
reference's Python bindings (``lazymat._core``, bindings/module.cpp:38-194)
on top of that C-ABI.
"""

__version__ = "0.1.0"
