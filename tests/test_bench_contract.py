"""bench.py contract on CPU: the reference arm's JSON line (keys, units, the
cpu_baseline and e2e objects; the live reference from baseline/_ref and the C
port), its torchrun behaviour (non-zero ranks exit silently) and the launcher's
hard failures (--gpus N without N GPUs, WORLD_SIZE != --gpus). The GPU arm is
exercised on the B200 (tests/test_gpu_bench.py and the driver)."""

import pytest

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env=None, extra_args=("--ref-impl", "port", "--cpu-seconds", "0.3"), rc=0):
    env = dict(os.environ, **(extra_env or {}))
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", *extra_args], capture_output=True, text=True, env=env,
                         timeout=600, cwd=ROOT)
    assert res.returncode == rc, res.stderr[-2000:]
    return [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]


def test_reference_arm_json_line():
    lines = _run()
    assert len(lines) == 1
    d = lines[0]
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "scaling", "vs_baseline",
              "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "rays/s" and d["value"] > 0
    assert d["higher_is_better"] is True and d["scaling"] == "weak" and d["vs_baseline"] is None
    assert {"workload", "envs_per_gpu", "cams", "resolution", "global_envs"} <= set(d["config"])
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert set(cb["split"]) >= {"render_only_mean", "render_plus_sensor_mean"}
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == "rays/s"
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_reference_arm_nonzero_rank_is_silent():
    assert _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"},
                extra_args=("--gpus", "2", "--ref-impl", "port", "--cpu-seconds", "0.3")) == []


@pytest.mark.skipif(not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "multidepth")),
                    reason="reference not installed in baseline/_ref")
def test_reference_arm_runs_the_live_reference():
    d = _run(extra_args=("--envs", "4", "--ref-impl", "live"))[0]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and "multidepth.render(backend='numba'" in cb["sample"]
    assert d["config"]["envs_per_gpu"] == 4 and d["value"] > 0


def test_launcher_fails_loudly():
    """--gpus 2 with no (or too few) GPUs and no share mode exits non-zero with a message;
    a torchrun world that disagrees with --gpus too."""
    bench = os.path.join(ROOT, "bench.py")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK",
                                                               "MDRT_BENCH_SHARE_GPU")}
    res = subprocess.run([sys.executable, bench, "--gpus", "2", "--steps", "1", "--warmup", "1"], capture_output=True,
                         text=True, env=env, timeout=300, cwd=ROOT)
    assert res.returncode != 0 and "bench.py:" in res.stderr
    env.update(RANK="0", WORLD_SIZE="2", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, bench, "--gpus", "1", "--steps", "1", "--warmup", "1"], capture_output=True,
                         text=True, env=env, timeout=300, cwd=ROOT)
    assert res.returncode == 2 and "WORLD_SIZE=2" in res.stderr


def test_config_dict_is_arm_independent_and_morton_is_a_permutation():
    """Both arms print config_dict(...) for the same run shape, so the driver can compare
    them key by key; the Z-order experiment renumbers envs without changing the set."""
    sys.path.insert(0, ROOT)
    import numpy as np
    import bench
    from paper_2602_03002_b200 import synth
    a = bench.config_dict("cfg2", 4096, 2, synth.config("cfg2", 8192))
    b = bench.config_dict("cfg2", 4096, 2, synth.config("cfg2", 4096))   # the reference arm's bounded sample
    assert a == b and a["global_envs"] == 8192 and a["terrain_tris"] == 259200
    w = synth.config("cfg2", 64)
    roots = w.roots.copy()
    bench.morton_order(w)
    assert sorted(map(tuple, w.roots)) == sorted(map(tuple, roots))
    assert not np.array_equal(w.roots, roots)
