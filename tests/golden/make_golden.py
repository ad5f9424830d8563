"""Generates tests/golden/oracle_golden.json from the CPU oracle.

The reference cannot be built here (Eigen missing), so these
fixtures are oracle outputs — pinned upstream by the reference's golden words
and known-answer tests (tests/test_oracle_golden.py). They freeze the
oracle bit-exactly (hex floats) and give the GPU parity tests fixed
expectations that do not depend on rebuilding anything.

    python tests/golden/make_golden.py      # rewrite the fixture
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def _hex(v):
    return [float(x).hex() for x in np.asarray(v, dtype=np.float64).reshape(-1)]


def compute(orc) -> dict:
    out = {}
    out["normals_seed1_len8"] = _hex(orc.RandomSource(1).normal_vector(8))
    out["normals_seed7_stream1_len5"] = _hex(orc.RandomSource(7, 1).normal_vector(5))
    out["derive_seed"] = [hex(orc.derive_seed(b, i)) for b, i in ((0, 0), (1, 0), (42, 7), (2 ** 63, 3))]
    # Haar n = 12, 6 probes, sides r r l r l r on x_t = data-stream normals
    op = orc.Operator("haar", n=12, seed=3)
    aux = orc.RandomSource(3, 1)
    ys = []
    for s in ("right", "right", "left", "right", "left", "right"):
        ys.append(op.probe(aux.normal_vector(12), s))
    out["haar12_seed3_probes"] = _hex(np.concatenate(ys))
    # Ginibre 10 x 7 sigma 0.5, sides r l r r l
    op = orc.Operator("ginibre", m=10, n=7, sigma=0.5, seed=4)
    aux = orc.RandomSource(4, 1)
    ys = []
    for s in ("right", "left", "right", "right", "left"):
        ys.append(op.probe(aux.normal_vector(7 if s == "right" else 10), s))
    out["ginibre10x7_seed4_probes"] = _hex(np.concatenate(ys))
    # config-1-shaped run at n = 64: alternating normalised power iteration
    n = 64
    op = orc.Operator("ginibre", m=n, n=n, sigma=1 / np.sqrt(n), seed=1)
    x1 = orc.RandomSource(1, 1).normal_vector(n)
    out["ginibre64_normalize_T20_final"] = _hex(op.run("normalize", "alternate", 20, x1, keep=False)[0])
    # config-2-shaped run at n = 128: tanh mix
    op = orc.Operator("haar", n=128, seed=2)
    x1 = orc.RandomSource(2, 1).normal_vector(128)
    x1 /= np.linalg.norm(x1)
    out["haar128_tanh_T25_final"] = _hex(op.run("tanh_mix", "right", 25, x1, keep=False)[0])
    # GOE n = 40 (inner sigma 1/sqrt n), 6 normalised steps
    op = orc.Operator("goe", n=40, sigma=1 / np.sqrt(40), seed=5)
    x1 = orc.RandomSource(5, 1).normal_vector(40)
    out["goe40_normalize_T6_final"] = _hex(op.run("normalize", "right", 6, x1, keep=False)[0])
    return out


def main():
    sys.path.insert(0, ROOT)
    from oracle import oracle as orc

    orc.build()
    with open(os.path.join(HERE, "oracle_golden.json"), "w") as f:
        json.dump(compute(orc), f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
