"""Generates tests/golden/chaos_envelope_config2.json: the CPU oracle's own
sensitivity envelope on BASELINE config 2 (SURVEY.md §7 hard part 6).

Config 2's map x_{t+1} = tanh(2 Q x_t) + 0.1 x_{t-1} is chaotic: rounding
differences grow roughly like e^{0.13 t}, so the 1e-9 iterate tolerance of the
north star cannot hold at late steps for ANY two correct implementations that
round differently. The envelope is measured oracle vs oracle: the same Haar
operator (reference draws, seed 2) run from x_1 and from x_1 perturbed by a
relative 1e-14 (about 50 ulps, i.e. more than the per-step rounding noise two
implementations accumulate), the per-iterate relative distance recorded for
t = 1..T+1. tests/test_gpu_fullsize.py holds the device to
max(1e-9, envelope[t]) at every iterate.

    python tests/golden/make_chaos_envelope.py      # rewrite the fixture (~1 min, 2 GB RAM)
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))

N, T, SEED, PERTURB = 1_000_000, 100, 2, 1e-14


def initial(orc):
    x1 = orc.RandomSource(SEED, 1).normal_vector(N)
    return x1 / np.linalg.norm(x1)


def compute(orc) -> dict:
    x1 = initial(orc)
    a = orc.Operator("haar", n=N, seed=SEED).run("tanh_mix", "right", T, x1, keep=True)
    xi = np.random.default_rng(11).standard_normal(N)
    b = orc.Operator("haar", n=N, seed=SEED).run("tanh_mix", "right", T, x1 * (1.0 + PERTURB * xi), keep=True)
    env = [float(np.linalg.norm(a[t] - b[t]) / np.linalg.norm(a[t])) for t in range(T + 1)]
    return {"n": N, "T": T, "seed": SEED, "perturbation": PERTURB, "map": "tanh_mix", "sides": "right",
            "envelope": env, "checksum_x_T1": float(a[T].sum())}


def main():
    sys.path.insert(0, ROOT)
    from oracle import oracle as orc

    orc.build()
    d = compute(orc)
    with open(os.path.join(HERE, "chaos_envelope_config2.json"), "w") as f:
        json.dump(d, f, indent=1)
    print("envelope t=1,25,50,75,100:", [d["envelope"][i] for i in (1, 25, 50, 75, 100)])


if __name__ == "__main__":
    main()
