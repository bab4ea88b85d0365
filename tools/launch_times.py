"""Summarise an `ncu --csv --metrics gpu__time_duration.sum[,...]` log: one line
per launch (kernel, metrics).  python tools/launch_times.py log.csv [regex]"""
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
hdr, cur, out = None, {}, []
for r in rows:
    if "Kernel Name" in r and "Metric Name" in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = (d["ID"], d["Kernel Name"])
    cur.setdefault(key, {})[d["Metric Name"]] = d["Metric Value"]
for (i, name), m in cur.items():
    if pat and not pat.search(name):
        continue
    short = re.sub(r"\(.*", "", name.replace("(anonymous namespace)::", "").replace("unnamed>::", ""))
    print(f"{int(i):4d} {short[:60]:60s} " + " ".join(f"{k.split('__')[-1]}={v}" for k, v in m.items()))
