"""bench.py's driver contract on the CPU side: the reference arm prints one JSON line with
the keys the driver reads, the same `config` object as the GPU arm, maps none of the
repo's product libraries, and `--gpus 2` spawns two ranks by itself (the GPU arm is
exercised on the B200 by the round-end bench)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run(args, timeout=600):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    return json.loads(lines[0])


def _check_reference_line(d):
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["unit"] == d["unit"]
    # the reference arm never maps the product library
    assert not any("libimconv" in p for p in d["native_libs"]), d["native_libs"]


def test_reference_arm_json_line():
    import bench
    from paper_2110_03901_b200.workloads import baseline_configs
    d = _run(["--impl", "reference", "--config", "cfg1", "--steps", "2", "--warmup", "1"])
    _check_reference_line(d)
    assert d["steps"] == 2
    # identical config object to what the GPU arm prints for the same workload and world
    assert d["config"] == bench.workload_config("cfg1", baseline_configs()["cfg1"], 1)
    from oracle import ref as R
    if R.available():
        assert d["cpu_baseline"]["kind"] == "reference"
        assert all(os.path.join("oracle", "_ref") in p for p in d["ref_shared_objects"])


def test_gpus_flag_spawns_ranks():
    """`--gpus 2` outside torchrun launches two ranks itself (gloo on a CPU host); rank 0
    alone prints, and n_gpus is the number of ranks that ran."""
    d = _run(["--impl", "reference", "--gpus", "2", "--config", "cfg1", "--steps", "1", "--warmup", "0"])
    _check_reference_line(d)
    assert d["n_gpus"] == 2
    assert d["config"]["parallelism"].startswith("dp2") and d["config"]["per_gpu_batch"] == 4


def test_workload_config_cfg4():
    import bench
    from paper_2110_03901_b200.workloads import baseline_configs
    layers = baseline_configs()["cfg4"]
    for world, per in ((1, 256), (2, 128), (8, 32)):
        c = bench.workload_config("cfg4", layers, world)
        assert c["global_batch"] == 256 and c["per_gpu_batch"] == per and c["layers"] == 53
        assert c["l2"].startswith("inputs larger than L2")
    assert bench.rotation_copies(baseline_configs()["cfg1"], 1) > 1


def test_gpu_arm_json_line():
    """The GPU arm on the B200 (cfg1, short): one JSON line with every key of the driver
    contract, the roofline / cpu_baseline / e2e / clocks objects, parity ok on the benchmarked
    outputs, kernel launches counted, the sweep and the serialised step both timed."""
    import pytest
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    d = _run(["--config", "cfg1", "--steps", "3", "--warmup", "3", "--no-traffic", "--cpu-sample", "1"])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
                "gpu_launches", "clocks", "parity"):
        assert key in d, key
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["gpu_launches"] > 0
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in d["roofline"], key
    assert 0 < d["roofline"]["frac"] < 1.5
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["parity"]["ok"] is True and d["parity"]["checked_images"] > 0
    assert d["run"]["layer_overlap"] is True and d["run"]["value_layers_serialized"] > 0
    assert "sm_mhz" in d["clocks"]


test_gpu_arm_json_line = __import__("pytest").mark.gpu(test_gpu_arm_json_line)
