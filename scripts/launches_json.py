"""Convert an ncu --metrics gpu__time_duration.sum --csv launch list into profiles/ JSON:
one record per launch plus a per-kernel share summary (the shares are what bench.py's live
timing must agree with; ncu's per-launch times are cold-cache and serialised)."""
import csv
import json
import sys
from collections import defaultdict


def main(src, dst):
    rows = list(csv.reader(open(src)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[i]
    ki, vi, gi, bi = (h.index(c) for c in ("Kernel Name", "Metric Value", "Grid Size", "Block Size"))
    unit_i = h.index("Metric Unit")
    launches = []
    for r in rows[i + 1:]:
        if len(r) != len(h):
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[unit_i], 1.0)
        launches.append({"id": int(r[0]), "kernel": r[ki], "grid": r[gi], "block": r[bi], "ns": v})
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for x in launches:
        name = x["kernel"].split("(")[0]
        tot[name] += x["ns"]
        cnt[name] += 1
    all_ns = sum(tot.values())
    summary = {k: {"launches": cnt[k], "total_ms": tot[k] / 1e6, "share": tot[k] / all_ns,
                   "mean_ms": tot[k] / cnt[k] / 1e6} for k in tot}
    json.dump({"summary": summary, "launches": launches}, open(dst, "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
