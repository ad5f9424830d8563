"""Per-source-line instruction counts and warp-stall samples of one kernel in
an ncu report captured with --import-source on (run here, on the CPU box):
    python tools/ncu_lines.py REPORT.ncu-rep LAUNCH_INDEX [TOP]"""
import collections, csv, io, subprocess, sys

rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
cur = h = None
agg = collections.defaultdict(lambda: [0, 0, ""])
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        h = r
        continue
    if h is None or len(r) != len(h):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    num = lambda x: int(x) if x.isdigit() else 0
    k = (cur, ln)
    agg[k][0] += num(r[h.index("Instructions Executed")])
    agg[k][1] += num(r[h.index("Warp Stall Sampling (All Samples)")])
    agg[k][2] = r[1][:90]
ti = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values()) or 1
print(f"instructions {ti}, stall samples {ts}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{100 * v[1] / ts:5.1f}% {v[0]:>10} {k[0]}:{k[1]}  {v[2]}")
