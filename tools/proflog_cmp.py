"""Compare HD_PROF_LOG per-launch logs of k_nt passes (fold2p / gin2p) by
column-count bucket: python tools/proflog_cmp.py LOG_A LOG_B [bucket]"""
import collections
import sys


def load(path):
    d = collections.defaultdict(lambda: [0.0, 0.0, 0, set()])
    for l in open(path):
        p = l.split()
        if p[0] not in ("fold2p", "gin2p"):
            continue
        kv = dict(x.split("=") for x in p[3:])
        rows = int(kv["nsub"]) * int(kv["rs"])
        key = (p[0], "m" if rows > 1.5e7 else "n", int(kv["C"]) // B * B)
        e = d[key]
        e[0] += float(p[1])
        e[1] += float(p[2])
        e[2] += 1
        e[3].add(f"{kv['rs']}/{kv['nst']}")
    return d


B = int(sys.argv[3]) if len(sys.argv) > 3 else 50
logs = [load(a) for a in sys.argv[1:3]]
keys = sorted(set(logs[0]) | set(logs[1]))
tot = [0.0, 0.0]
for k in keys:
    a, b = logs[0].get(k), logs[1].get(k)
    ra = a[0] / a[1] / 1e9 if a else 0
    rb = b[0] / b[1] / 1e9 if b else 0
    tot[0] += a[1] if a else 0
    tot[1] += b[1] if b else 0
    print(f"{k[0]:7s} {k[1]} C{k[2]:4d}+  A {a[1] if a else 0:8.2f} ms {ra:5.2f} TB/s {sorted(a[3]) if a else ''}"
          f"   B {b[1] if b else 0:8.2f} ms {rb:5.2f} TB/s {sorted(b[3]) if b else ''}")
print(f"total A {tot[0]:.1f} ms  B {tot[1]:.1f} ms")
