python - <<'PY'
import os, sys, time, subprocess, json
for env in ({}, {"FEWHA_WFS_BATCH_MINB": "3"}, {"FEWHA_GATHER_MINB": "2"}, {"FEWHA_GATHER_MINB": "4"}):
    e = dict(os.environ); e.update(env)
    out = subprocess.run([sys.executable, "bench.py", "--steps", "20", "--warmup", "3", "--no-configs", "--no-cpu"], env=e, capture_output=True, text=True).stdout
    j = json.loads(out.strip().splitlines()[-1]); b = j["batch64"]
    print(env, "b64 ms", b["ms_per_step"], "1x64", b["ms_per_step_1x64"], {k: v["launch_ms"] for k, v in b["roofline"]["functions"].items()}, flush=True)
PY
