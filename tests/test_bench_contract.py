"""The bench.py reference arm (the oracle on the host cores, this tier's `--impl reference`) keeps
the driver's JSON contract; it runs on CPU, so it is checked here every round."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra=None):
    env = dict(os.environ)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "3",
                           "--warmup", "3"], capture_output=True, text=True, cwd=ROOT, env=env, timeout=600)


def test_reference_arm_json_line():
    r = _run()
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        metric = json.load(f)["metric"]
    assert d["impl"] == "reference" and d["metric"] == metric
    assert d["unit"] == "surfaces/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["vs_baseline"] is None and d["data"] == "synthetic"
    assert d["config"]["workload"].startswith("C3")
    # the reference arm reports our arm's config for the same world size (the driver compares them)
    import importlib.util
    spec = importlib.util.spec_from_file_location("_bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    assert d["config"] == bench.workload_config("C3", 1, 0)
    assert d["reference_windows_per_step"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] == d["value"] and cb["cores"] >= 1 and cb["sample"]


def test_reference_arm_does_not_map_the_product_library():
    d = json.loads(_run().stdout.strip().splitlines()[-1])
    assert not any("libieds" in p for p in d["repo_native_libs_mapped"]), d["repo_native_libs_mapped"]


def test_bare_gpus_2_relaunches_two_ranks():
    """`bench.py --gpus 2` without torchrun re-runs itself as 2 ranks (torch.distributed.run on
    127.0.0.1): one JSON line, from rank 0, reporting the real world size and the N > 1 config
    (C4: BASELINE configs[3], 16k windows sharded)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "3", "--warmup", "3"], capture_output=True, text=True, cwd=ROOT, timeout=600,
                       env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["config"]["workload"].startswith("C4") and d["scaling"] == "strong"


def test_reference_arm_other_ranks_exit_quietly():
    r = _run({"RANK": "1", "LOCAL_RANK": "1", "WORLD_SIZE": "2"})
    assert r.returncode == 0, r.stderr[-2000:]
    assert not r.stdout.strip()


@pytest.mark.gpu
def test_ours_json_line_contract():
    """Our arm's line carries every key of the driver contract (short run, rows skipped)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3", "--no-exact",
                        "--no-f1", "--no-f3", "--no-f4", "--no-c2", "--no-c5", "--no-c4-r1", "--no-latency"],
                       capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.strip()][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["scaling"] == "weak"
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] <= 1.5
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["gpu_launches"] == 2 * d["steps"]   # one frame + one window launch per 1000-window step
    import importlib.util
    spec = importlib.util.spec_from_file_location("_bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    # the reference arm reports this same config (test_reference_arm_json_line)
    assert d["config"] == bench.workload_config("C3", 1, 0, events_per_gpu=d["config"]["events_per_gpu"])
    assert d["config"]["events_per_gpu"] == 75_000_000
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@pytest.mark.gpu
def test_ours_two_ranks_code_path():
    """The N > 1 path of our arm (`bench.py --gpus 2` relaunching under torchrun, C4 sharded,
    cross-rank digest check), exercised on a one-GPU box: IEDS_BENCH_SHARE_GPU=1 puts both ranks
    on cuda:0 with the gloo backend.  A code-path check only -- the numbers are not a measurement."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["IEDS_BENCH_SHARE_GPU"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--windows", "64", "--c5-windows", "32", "--no-exact", "--no-f1", "--no-c2", "--no-e2e",
                        "--no-cpu-baseline"], capture_output=True, text=True, cwd=ROOT, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["config"]["workload"].startswith("C4")
    assert d["config"]["windows_total"] == 64 and d["config"]["windows_per_gpu"] == 32
    assert d["dist"]["world_size"] == 2 and d["dist"]["shared_gpu_code_path_check"] is True
    assert d["cross_rank_check"]["match"] is True and d["cross_rank_check"]["windows_checked"] == 6
    assert d["c5_burst"]["windows_total"] == 32 and d["c5_burst"]["scaling"] == "strong"
    assert d["c3_weak_scaling"]["scaling"] == "weak" and d["c3_weak_scaling"]["windows_per_gpu"] == 32
    assert d["gpu_launches"] == 2 * d["steps"]
