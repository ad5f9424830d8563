"""The `lazymat bench` front-end (tools/lazymat_cli.cpp:384-494 mirrored in
paper_2101_07464_b200/lazymat/cli.py): usage errors and exit codes on CPU;
the CSV / manifest / slope output, the resource-cap exit and manifest replay
on the GPU (test_cli.cpp's end-to-end checks restated)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cli(*args, cwd=None):
    return subprocess.run([sys.executable, "-m", "paper_2101_07464_b200.lazymat.cli", *args], capture_output=True,
                          text=True, cwd=cwd or ROOT, timeout=900)


def test_usage_errors_exit_2(tmp_path):
    assert cli("--out", str(tmp_path)).returncode == 2                       # no subcommand
    assert cli("--out", str(tmp_path), "bench", "--backend", "gpu").returncode == 2  # not a choice
    assert cli("--out", str(tmp_path), "bench", "--reps", "x").returncode == 2
    r = cli("--out", str(tmp_path), "--from-manifest", str(tmp_path / "missing.json"))
    assert r.returncode == 2 and "cannot read manifest" in r.stderr
    (tmp_path / "m.json").write_text(json.dumps({"subcommand": "ista", "config": {}}))
    r = cli("--out", str(tmp_path), "--from-manifest", str(tmp_path / "m.json"))
    assert r.returncode == 2 and "unknown subcommand" in r.stderr
    r = cli("--out", str(tmp_path), "--version")
    assert r.returncode == 0 and r.stdout.strip() == "0.1.0"


def test_loglog_fit_and_grid():
    sys.path.insert(0, ROOT)
    from paper_2101_07464_b200.lazymat import cli as c

    assert c.power_grid(512, 4096) == [512, 1024, 2048, 4096]
    assert abs(c.fit_loglog([1, 2, 4, 8], [3, 6, 12, 24]) - 1.0) < 1e-12
    assert abs(c.fit_loglog([1, 2, 4], [1, 4, 16]) - 2.0) < 1e-12
    assert c.median_of([3.0, 1.0, 2.0, 10.0]) == 2.5
    with pytest.raises(c.UsageError):
        c.power_grid(8, 4)


@pytest.mark.gpu
def test_bench_csv_manifest_slopes_and_replay(tmp_path, lm):
    out = tmp_path / "run"
    r = cli("--out", str(out), "bench", "--backend", "both", "--nmin", "256", "--nmax", "1024", "-T", "8",
            "--reps", "1")
    assert r.returncode == 0, r.stderr
    assert "slope(backend=hd, axis=n)" in r.stdout and "slope(backend=direct, axis=n)" in r.stdout
    lines = (out / "bench.csv").read_text().splitlines()
    assert lines[0] == "backend,n,T,median_ms"
    rows = [ln.split(",") for ln in lines[1:]]
    assert [(b, int(n), int(t)) for b, n, t, _ in rows] == [(b, n, 8) for b in ("hd", "direct")
                                                             for n in (256, 512, 1024)]
    assert all(float(ms) > 0 for *_, ms in rows)
    man = json.loads((out / "bench_manifest.json").read_text())
    assert man["subcommand"] == "bench" and man["deterministic"] is False and man["outputs"] == ["bench.csv"]
    assert man["config"]["backend"] == "both" and man["config"]["T"] == 8 and len(man["slopes"]) == 2
    # replay: the same configuration, the same points
    out2 = tmp_path / "replay"
    r = cli("--out", str(out2), "--from-manifest", str(out / "bench_manifest.json"))
    assert r.returncode == 0, r.stderr
    rows2 = [ln.split(",")[:3] for ln in (out2 / "bench.csv").read_text().splitlines()[1:]]
    assert rows2 == [row[:3] for row in rows]
    # T sweep at fixed n
    r = cli("--out", str(tmp_path / "t"), "bench", "--fix-n", "--fixed-n", "2048", "--sweep-T", "4", "8", "16",
            "--reps", "1")
    assert r.returncode == 0 and "axis=T" in r.stdout
    # the dense backend beyond the oracle cap: resource-cap exit
    r = cli("--out", str(tmp_path / "cap"), "bench", "--backend", "direct", "--nmin", "4096", "--nmax", "4096",
            "-T", "4", "--reps", "1", "--dim-cap", "2048")
    assert r.returncode == 4 and "resource cap" in r.stderr
