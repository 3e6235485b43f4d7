"""A/B of plan knobs on the batch-64 step (profiling aid)."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
envs = [json.loads(a) for a in sys.argv[1:]] or [{}]
for env in envs:
    e = dict(os.environ)
    e.update(env)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "20", "--warmup", "3", "--no-configs",
                        "--no-cpu"], env=e, capture_output=True, text=True)
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    if not lines:
        print(env, "FAILED", p.stderr[-500:], flush=True)
        continue
    j = json.loads(lines[-1])
    b = j["batch64"]
    print(env, "lat", j["latency"]["p50_ms"], "b64", b["ms_per_step"], "1x64", b["ms_per_step_1x64"],
          {k: v["launch_ms"] for k, v in b["roofline"]["functions"].items()}, flush=True)
