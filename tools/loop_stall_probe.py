"""Is the c5 loop's run-to-run spread (bench.py --loop: 1.5 ms/step in most runs, 2.6-5.5 in a few) caused
by the nvidia-smi clock sampler running next to the loop's host work (prunes, re-captures)?  Runs
bench.run_loop alternately with the sampler and with a no-op in its place, and prints ms/step of each run.
usage (GPU box, repo root): python tools/loop_stall_probe.py [REPS] [--per-set]"""
import sys

sys.path.insert(0, '.')
import bench  # noqa: E402


class NoClock:
    def __init__(self, index):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        pass

    def summary(self):
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}


class Args:
    config = "c5"
    steps = 100
    warmup = 3
    prune_every = 15
    per_set = "--per-set" in sys.argv
    targets = "u8"
    no_spatial_order = False


reps = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 4
real = bench.ClockSampler
for r in range(reps):
    for name, cls in (("sampler", real), ("none", NoClock)):
        bench.ClockSampler = cls
        out = bench.run_loop(Args)
        print(r, name, out["ms_per_step"], out["clocks"].get("samples"), flush=True)
