"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py full  gpurun_out/prof.ncu-rep  profiles/rNN_full.json
    python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/rNN_launches.json
"""
import collections
import csv
import io
import json
import subprocess
import sys


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    keys = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
            "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct"]
    res = []
    for r in rows[2:]:
        d = {k: r[h.index(k)] for k in keys if k in h}
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(r[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        d["top_stalls_pct"] = {k: round(100 * v / tot, 1) for v, k in sorted(stalls, reverse=True)[:6]}
        units = {k: r[h.index(k)] for k in keys if k in h}
        d["units"] = {k: rows[1][h.index(k)] for k in keys if k in h}
        try:
            us = float(d["gpu__time_duration.sum"])
            if d["units"].get("gpu__time_duration.sum") == "nsecond":
                us /= 1e3
            sc = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}
            b = (float(d["dram__bytes_read.sum"]) * sc[d["units"]["dram__bytes_read.sum"]] +
                 float(d["dram__bytes_write.sum"]) * sc[d["units"]["dram__bytes_write.sum"]])
            d["dram_GBps"] = b / (us * 1e-6) / 1e9
            d["dram_bytes"] = b
        except Exception:
            pass
        res.append(d)
    json.dump(res, open(out, "w"), indent=1)
    for d in res:
        print(d.get("Kernel Name"), d.get("gpu__time_duration.sum"), round(d.get("dram_GBps", 0)), d["top_stalls_pct"])


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    res = {k: {"launches": c, "total_us": round(t, 1), "avg_us": round(t / c, 2), "share": round(t / tot, 4)}
           for k, (c, t) in agg.items()}
    json.dump(res, open(out, "w"), indent=1)
    for k, v in res.items():
        print(f"{k:40s} {v}")


def traffic(full_json, out, t=91, n=1_000_000):
    """DRAM bytes of the captured config-2 probe t vs the library's algorithmic
    bytes for it (hd_lib.cu LaunchScope accounting, fp64):
      k_dots   8 n (t + 1): fold chain (t-1 columns) + its pending column + x
                            (the mix column was written by the previous OTHER)
      FOLD     8 n (t + 1): fold chain (t-1 columns) + x + the new column
      OTHER    8 n (t + 3): other chain (t columns) + output + next mix column
                            + x_{t-1} (tanh mix)"""
    alg = {"dots": 8 * n * (t + 1), "fold": 8 * n * (t + 1), "other": 8 * n * (t + 3),
           # two-pass pass: other panel t + fold panel t - 1
           # columns, new fold column, x_t, x_{t+1}, x_{t-1}, next mix column
           "haar2p": 8 * n * (2 * t + 4)}
    kind = {"k_dots": "dots", "k_apply<double, 0>": "fold", "k_apply<double, 1>": "other",
            "k_haar2p<double>": "haar2p"}
    res = {}
    for d in json.load(open(full_json)):
        name = d.get("Kernel Name", "")
        for key, k in kind.items():
            # the capture holds probes t and t + 1: keep the first (probe t), whose bytes alg[k] describes
            if key in name and "dram_bytes" in d and k not in res:
                us = float(d["gpu__time_duration.sum"]) / (1e3 if d["units"]["gpu__time_duration.sum"] == "nsecond" else 1)
                res[k] = {"probe_t": t, "dram_bytes": d["dram_bytes"], "alg_bytes": alg[k],
                          "ratio": d["dram_bytes"] / alg[k], "ncu_us": us,
                          "source": f"{full_json} (ncu --set full, cold cache, serialised)"}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    {"full": full, "launches": launches, "traffic": traffic}[sys.argv[1]](sys.argv[2], sys.argv[3])
