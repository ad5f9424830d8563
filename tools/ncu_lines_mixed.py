"""Per-CUDA-source-line warp-stall samples from an ncu report's mixed
cuda,sass source page (ncu -i REP --page source --csv --print-source cuda,sass).
Usage: python tools/ncu_lines_mixed.py page.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, out = "", None, []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0]:
        s = int(r[hdr.index("# Samples")] or 0)
        if s:
            st = {hdr[i]: int(r[i]) for i in range(len(hdr)) if hdr[i].startswith("stall_")
                  and "Not Issued" not in hdr[i] and r[i] not in ("", "0")}
            out.append((s, f"{fname}:{r[0]}", r[1].strip()[:80], st))
tot = sum(o[0] for o in out)
print("total samples", tot)
for s, loc, src, st in sorted(out, reverse=True)[:top]:
    t3 = ", ".join(f"{k[6:]} {v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3])
    print(f"{s:7d} {100 * s / tot:5.1f}% {loc:22s} {src:80s} {t3}")
