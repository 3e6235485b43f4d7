"""Per-kernel-function DRAM bytes per launch from ncu launch lists.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none -s <skip> -c <one frame> --csv --log-file <csv> \
        python tools/profile_frame.py [--batch 64]
    python tools/dram_traffic.py <key>=<csv> ...   -> profiles/dram_traffic.json

ncu replays each launch with its caches flushed, so these are cold-cache bytes
(read + write) per launch, averaged over the function's launches in the frame;
bench.py puts the dominant function's figure in roofline.traffic.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def parse(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
    per = {}
    for r in rows[1:]:
        name = r[ix["Kernel Name"]].split("<")[0].split("(")[0].replace("void ", "").strip().split("::")[-1]
        key = (r[ix["ID"]], name)
        m, u, v = r[ix["Metric Name"]], r[ix["Metric Unit"]], r[ix["Metric Value"]]
        v = float(v.replace(",", ""))
        e = per.setdefault(key, {})
        if m.startswith("dram__bytes"):
            e["dram"] = e.get("dram", 0.0) + v * UNIT.get(u, 1)
        elif m == "gpu__time_duration.sum":
            e["us"] = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
    funcs = {}
    for (_, name), e in per.items():
        f = funcs.setdefault(name, {"launches": 0, "dram": 0.0, "us": 0.0})
        f["launches"] += 1
        f["dram"] += e.get("dram", 0.0)
        f["us"] += e.get("us", 0.0)
    return {k: int(v["dram"] / v["launches"]) for k, v in funcs.items()}, funcs


if __name__ == "__main__":
    out_path = os.path.join(ROOT, "profiles", "dram_traffic.json")
    old = json.load(open(out_path)) if os.path.exists(out_path) else {}
    out = {k: v for k, v in old.items() if not isinstance(v, dict) or any(x.startswith("k_") for x in v)}
    for arg in sys.argv[1:]:
        key, path = arg.split("=", 1)
        out[key], funcs = parse(path)
        out[key + "_source"] = os.path.relpath(path, ROOT)
        print(key, {k: (v["launches"], round(v["us"], 1), int(v["dram"] / v["launches"])) for k, v in funcs.items()})
    json.dump(out, open(out_path, "w"), indent=1)
