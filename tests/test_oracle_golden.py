"""Pin the CPU oracle (oracle/oracle.c) against the reference's own outputs.

The goldens under tests/golden/ were produced by running the live reference
(`multidepth`, numba backend) on float32-representable inputs
(tests/golden/make_golden.py). The oracle restates the same f64 algorithm,
so it must reproduce them bit-for-bit (render, rng, latency, downsample) or to
within libm last-ulp effects (noise: log/cos).
"""

import glob
import os

import numpy as np
import pytest

import casefile
from conftest import GOLDEN

RENDER_CASES = sorted(glob.glob(os.path.join(GOLDEN, "render_*.npz")))


def oracle_render(oracle, case, **kw):
    sc = oracle.OracleScene(casefile.bodies(case), casefile.terrain(case), casefile.cameras_dicts(case))
    r = casefile.rand(case)
    n = int(case["num_envs"])
    bp, bq = case["body_pos"], case["body_rot"]
    if bp.shape[1] == 0:
        bp, bq = np.zeros((n, 0, 3)), np.zeros((n, 0, 4))
    return sc.render(bp, bq, rand_pos=None if r is None else r[0], rand_rot=None if r is None else r[1],
                     fov_delta=None if r is None else r[2], early_termination=bool(case["early"]), **kw)


def test_golden_cases_present():
    names = {os.path.basename(p) for p in RENDER_CASES}
    for need in ("render_cfg1.npz", "render_flat.npz", "render_miss.npz", "render_parented.npz",
                 "render_rand_camrand.npz", "render_cfg2_slice.npz"):
        assert need in names


@pytest.mark.parametrize("path", RENDER_CASES, ids=lambda p: os.path.basename(p)[7:-4])
def test_oracle_render_matches_reference(oracle, path):
    case = casefile.load(path)
    out = oracle_render(oracle, case, threads=2)
    ref = case["out"]
    assert out.shape == ref.shape
    diff = np.abs(out.astype(np.float64) - ref.astype(np.float64))
    # same f64 algorithm, same operation order, no FMA contraction: bit-exact
    assert np.array_equal(out, ref), f"max diff {diff.max()}, equal fraction {np.mean(out == ref)}"


def test_oracle_render_thread_count_invariant(oracle):
    case = casefile.load(os.path.join(GOLDEN, "render_cfg2_slice.npz"))
    a = oracle_render(oracle, case, threads=1)
    b = oracle_render(oracle, case, threads=4)
    assert np.array_equal(a, b)


def test_oracle_counts_visits(oracle):
    case = casefile.load(os.path.join(GOLDEN, "render_cfg1.npz"))
    ctr = np.zeros(2, np.int64)
    oracle_render(oracle, case, counters=ctr)
    rays = case["out"].size
    # reference BVH: every ray visits all 30 link roots plus the terrain path
    assert ctr[0] / rays > 30 and ctr[1] > 0


def test_oracle_analytic_flat(oracle):
    case = casefile.load(os.path.join(GOLDEN, "render_flat.npz"))
    out = oracle_render(oracle, case)[0, 0]
    assert out[3, 4] == pytest.approx(1.0, abs=1e-6)
    _, scale = oracle.ray_grid(9, 7, 70.0, 55.0)
    assert np.allclose(out, scale, atol=1e-5)


def test_oracle_miss_is_dmax(oracle):
    case = casefile.load(os.path.join(GOLDEN, "render_miss.npz"))
    assert np.all(oracle_render(oracle, case) == np.float32(3.5))


@pytest.fixture(scope="module")
def sens():
    return casefile.load(os.path.join(GOLDEN, "sensor.npz"))


def test_oracle_rng_bit_exact(oracle, sens):
    for seed, name, val in zip(sens["keys_seed"], ["sensor", "sensor", "latency", "a-much-longer-stream-name"],
                               sens["keys_val"]):
        assert oracle.stream_key(int(seed), name) == int(val)
    key = oracle.stream_key(5, "demo")
    c = sens["rng_counters"]
    assert np.array_equal(oracle.uniform(key, c[:, 0], c[:, 1]), sens["rng_uniform"])
    # Box-Muller through libm log/cos: allow one f64 ulp
    assert np.allclose(oracle.normal(key, c[:, 0], c[:, 1]), sens["rng_normal"], rtol=4e-16, atol=0)


def test_oracle_noise_matches_reference(oracle, sens):
    out = oracle.apply_noise_dropout(sens["depth"], noise_scale=0.1, dropout_p=0.05, seed=7,
                                     d_max=sens["d_max"], step=3)
    ref = sens["out_s3"]
    # dropout mask is integer arithmetic: exact
    drop_ref = ref == np.float32(8.0)
    assert np.mean(out == ref) > 0.9999
    assert np.max(np.abs(out.astype(np.float64) - ref)) <= 1e-5
    ulps = np.abs(out.view(np.int32).astype(np.int64) - ref.view(np.int32).astype(np.int64))
    assert ulps.max() <= 1
    out2 = oracle.apply_noise_dropout(sens["depth"], noise_scale=0.2, dropout_p=0.3, seed=2,
                                      d_max=sens["d_max"], step=0, dropout_fill=0.25)
    assert np.mean(out2 == sens["out_fill_s0"]) > 0.9999
    del drop_ref


def test_oracle_noise_env_offset_slices(oracle, sens):
    full = sens["out_s3_full8"]
    part = oracle.apply_noise_dropout(sens["depth"][2:4], noise_scale=0.1, dropout_p=0.05, seed=7,
                                      d_max=sens["d_max"], step=3, env_offset=6)
    assert np.array_equal(part, oracle.apply_noise_dropout(
        np.concatenate([sens["depth"], sens["depth"]]), noise_scale=0.1, dropout_p=0.05, seed=7,
        d_max=sens["d_max"], step=3)[6:8])
    assert np.mean(part == full[6:8]) > 0.9999


def test_oracle_latency_selection_bit_exact(oracle, sens):
    dt = float(sens["latency_dt"])
    cap = int(sens["latency_capacity"])
    delays = sens["delays"]
    for s, ref in enumerate(sens["latency_sel"]):
        ks = list(range(max(0, s - cap + 1), s + 1))
        times = np.array([k * dt for k in ks])
        idx = oracle.frame_select(times, s * dt, delays)
        assert np.array_equal(np.array(ks)[idx], ref), f"step {s}"


def test_oracle_latencies_and_downsample(oracle, sens):
    assert np.array_equal(oracle.sample_latencies(0.1, 5, 100, episode=2), sens["latencies_ep2"])
    assert np.array_equal(oracle.downsample_min(sens["ds_in"], 5), sens["ds_out"])


def test_oracle_rsm_matches_reference(oracle, sens):
    """Random side masking (perception.py:150-202): modes and fills bit-exact."""
    assert np.array_equal(oracle.rsm_sample_modes((0.6, 0.3, 0.1), 3, 64, 2, episode=1), sens["rsm_modes_stones"])
    out = oracle.rsm_apply(sens["rsm_depth"], sens["rsm_modes"], f_small=0.125, f_large=0.25, fill_low=0.3,
                           fill_high=None, seed=3, d_max=[6.0, 8.0], step=5)
    assert np.array_equal(out, sens["rsm_out_s5"])
    out2 = oracle.rsm_apply(sens["rsm_depth"], sens["rsm_modes"], f_small=0.1, f_large=0.3, fill_low=0.3,
                            fill_high=4.0, seed=4, d_max=[6.0, 8.0], step=0)
    assert np.array_equal(out2, sens["rsm_out2_s0"])
