"""Run bench.py on every BASELINE config (default flags, 1 GPU) and collect the JSON lines into one file:
python tools/config_sweep.py OUT.json [--steps K]"""
import json
import subprocess
import sys

out = sys.argv[1]
steps = sys.argv[sys.argv.index("--steps") + 1] if "--steps" in sys.argv else "20"
res = {}
for cfg in ("c1", "c2", "c3", "c4", "c5"):
    p = subprocess.run([sys.executable, "bench.py", "--config", cfg, "--steps", steps, "--warmup", "5",
                        "--no-cpu-baseline"], capture_output=True, text=True)
    line = [l for l in p.stdout.splitlines() if l.startswith("{")]
    res[cfg] = json.loads(line[-1]) if line else {"error": p.stderr[-2000:]}
    r = res[cfg]
    print(cfg, r.get("value"), (r.get("e2e") or {}).get("value"), (r.get("local_full") or {}).get("ratio"), flush=True)
for per_set in (False, True):
    args = [sys.executable, "bench.py", "--config", "c5", "--loop", "--steps", "100", "--warmup", "3"]
    if per_set:
        args.append("--per-set")
    p = subprocess.run(args, capture_output=True, text=True)
    line = [l for l in p.stdout.splitlines() if l.startswith("{")]
    key = "c5_loop_per_set" if per_set else "c5_loop_union"
    res[key] = json.loads(line[-1]) if line else {"error": p.stderr[-2000:]}
    print(key, res[key].get("value"), flush=True)
json.dump(res, open(out, "w"), indent=1)
