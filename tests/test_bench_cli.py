"""bench.py's launch contract on CPU (no GPU needed): the rank-count check,
and the reference arm (oracle/_ref on the host cores) printing the driver's
JSON line for a multi-GPU configuration -- the z-box weak-scaling problem at
the GPU run's partition, its step a bounded sample, its value the
extrapolated full solve."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env=None, timeout=600):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          cwd=ROOT, env=e, timeout=timeout)


def test_world_size_must_match_gpus():
    r = run(["--gpus", "2", "--steps", "1"], env={"WORLD_SIZE": "1"})
    assert r.returncode != 0 and "--gpus 2 but launched as 1 ranks" in r.stderr


def test_reference_arm_multi_gpu_line():
    r = run(["--impl", "reference", "--gpus", "2", "--nd", "16", "--steps", "2", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["unit"] == "s" and not d["higher_is_better"]
    assert d["config"]["workload"] == "poisson7_16x16x32_weak" and d["config"]["unknowns"] == 16 * 16 * 32
    assert d["iterations"] and d["value"] > 0 and d["full_solve_s"] is not None
    # the step is the bounded sample (3 iterations), the value the full solve
    assert abs(d["value"] - d["ms_per_iter"] * 1e-3 * d["iterations"]) < 1e-12
    assert d["ms_per_step"] < 1e3 * d["value"]
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] == 2
    assert d["e2e"] == {"value": d["value"], "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_quietly():
    r = run(["--impl", "reference", "--gpus", "2", "--nd", "16", "--steps", "1"], env={"WORLD_SIZE": "2", "RANK": "1"})
    assert r.returncode == 0 and r.stdout.strip() == ""
