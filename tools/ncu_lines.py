"""Aggregate ncu source-page (cuda,sass) warp-stall samples per CUDA source line."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
f = None; res = []; hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr and r and r[0] and len(r) == len(hdr):
        try:
            v = int(r[4] or 0)
        except ValueError:
            continue
        res.append((v, f, r[0], r[1].strip()[:110]))
tot = sum(x[0] for x in res)
print("total samples", tot)
for v, fn, ln, src in sorted(res, reverse=True)[:n]:
    print(f"{v:6d} {100*v/max(tot,1):5.1f}% {fn}:{ln} {src}")
