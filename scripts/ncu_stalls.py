"""Warp-stall breakdown of an ncu --set full report (source page, SASS): stall reasons in % of samples,
samples by opcode, and the hottest instructions with their neighbourhood.  Usage: ncu_stalls.py REP [N]."""
import csv
import io
import json
import subprocess
import sys
from collections import Counter


def main(rep, ntop=12):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, data = rows[1], rows[2:]
    si, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    data = [r for r in data if len(r) == len(h) and r[si].isdigit()]
    tot = sum(int(r[si]) for r in data)
    reasons = Counter()
    for j, name in enumerate(h):
        if name.startswith("stall_") and "(Not Issued)" not in name:
            reasons[name] = sum(int(r[j]) for r in data if r[j].isdigit())
    ops = Counter()
    for r in data:
        t = r[src].strip().split()
        o = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
        ops[o.split(".")[0]] += int(r[si])
    top = sorted(range(len(data)), key=lambda i: -int(data[i][si]))[:ntop]
    hot = []
    for i in top:
        ctx = [data[k][src].strip()[:60] for k in range(max(0, i - 3), i + 1)]
        why = {h[j]: int(data[i][j]) for j in range(len(h)) if h[j].startswith("stall_") and "(Not" not in h[j]
               and data[i][j].isdigit() and int(data[i][j]) > 0.1 * int(data[i][si])}
        hot.append({"pct": round(100 * int(data[i][si]) / tot, 2), "context": ctx, "stalls": why})
    print(json.dumps({"samples": tot, "stall_reasons_pct": {k: round(100 * v / tot, 2) for k, v in reasons.most_common() if v},
                      "opcodes_pct": {k: round(100 * v / tot, 2) for k, v in ops.most_common(12)}, "hot": hot}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12)
