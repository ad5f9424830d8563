"""The C-ABI from a C++ host (north star: "the host side is C++ calling CUDA
through a thin C-ABI"): examples/b200_probe_operator.hpp adapts hd.h to the
reference's ProbeOperator shape; examples/cabi_demo.cpp drives config 2's
dynamics probe by probe and as one hd_run. Compiled with g++ here; run on
the GPU."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2101_07464_b200", "lib")


def _compile(out):
    subprocess.run(["g++", "-O2", "-std=c++17", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    "-I", os.path.join(ROOT, "examples"), os.path.join(ROOT, "examples", "cabi_demo.cpp"),
                    "-L", LIBDIR, "-lhd_b200", f"-Wl,-rpath,{LIBDIR}", "-o", out], check=True)


def test_cpp_host_compiles_and_links_against_the_cabi(lm, tmp_path):
    exe = str(tmp_path / "cabi_demo")
    _compile(exe)
    assert os.path.exists(exe)
    # plain C can include the header too (no C++ or CUDA types in the boundary)
    src = tmp_path / "c_include.c"
    src.write_text('#include "hd.h"\nint main(void) { return hd_version() == 0; }\n')
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), str(src), "-L", LIBDIR,
                    "-lhd_b200", f"-Wl,-rpath,{LIBDIR}", "-o", str(tmp_path / "c_include")], check=True)


@pytest.mark.gpu
def test_cpp_host_runs_config2_dynamics(lm, tmp_path):
    exe = str(tmp_path / "cabi_demo")
    _compile(exe)
    r = subprocess.run([exe, "200000", "20"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["isometry_err"] < 1e-12 and d["routes_rel_diff"] < 1e-12 and d["budget_exception"]
