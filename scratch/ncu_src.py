"""Per CUDA source line: warp-stall samples and warp-level instructions executed (ncu source page)."""
import csv, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
f = None; hdr = None; res = {}
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        f = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr and r and r[0] and len(r) == len(hdr) and r[0].isdigit():
        try:
            samp = int(r[4] or 0); ins = int(r[7] or 0)
        except ValueError:
            continue
        key = (f, int(r[0]))
        a = res.setdefault(key, [0, 0, r[1].strip()[:100]]); a[0] += samp; a[1] += ins
ts = sum(v[0] for v in res.values()); ti = sum(v[1] for v in res.values())
print(f"total samples {ts}, warp instructions {ti}")
for (fn, ln), (s, i, src) in sorted(res.items(), key=lambda kv: -kv[1][1])[:n]:
    print(f"{i:10d} {100*i/max(ti,1):5.1f}% ins {100*s/max(ts,1):5.1f}% smp {fn}:{ln} {src}")
