"""Per-source-line warp-stall breakdown of an ncu report (source page, cuda+sass).

    python tools/diag/ncu_lines_stalls.py REPORT FILE LINE_FROM LINE_TO
"""
import collections
import csv
import subprocess
import sys

rep, fname, l0, l1 = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
agg = collections.defaultdict(collections.Counter)
src = {}
f = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) == len(hdr) and r[0].isdigit() and f == fname and l0 <= int(r[0]) <= l1:
        d = dict(zip(hdr, r))
        ln = int(r[0])
        src.setdefault(ln, r[1].strip()[:70])
        for k in hdr:
            if (k.startswith("stall_") and "(Not" not in k) or k in ("L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal",
                                                                      "Instructions Executed"):
                try:
                    agg[ln][k] += int(float(d[k] or 0))
                except ValueError:
                    pass
for ln in sorted(agg):
    c = agg[ln]
    top = [(k[6:], v) for k, v in c.most_common() if k.startswith("stall") and v > 0][:4]
    tot = sum(v for k, v in c.items() if k.startswith("stall"))
    print(f"{ln:5d} {tot:6d} inst {c['Instructions Executed']:6d} wf {c['L1 Wavefronts Shared']:6d}/{c['L1 Wavefronts Shared Ideal']:6d} "
          f"{top}  | {src.get(ln, '')}")
