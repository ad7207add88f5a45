"""Tier pipeline: the theta solver / schedule model against the reference's acceptance
values (test_acceptance.py c05, c06) on CPU, and the pinned-host -> HBM stream with the
INT4 split on the GPU."""

from __future__ import annotations

import dataclasses

import numpy as np
import pytest

from paper_2506_20187_b200.tier import LayerLoad, PipelineParams, build_schedule, compare_modes, solve_theta


def test_c05_theta_solver():
    params = PipelineParams(compute_ms=10.0, overhead_ms=4.0, bw_hot_warm=8.0, compress_ratio=0.25,
                            decompress_rate=32.0)
    sol = solve_theta(64.0, params)
    assert sol.feasible and abs(sol.theta - 0.25) <= 1e-9
    hidden = solve_theta(8.0, dataclasses.replace(params, overhead_ms=0.0))
    assert hidden.theta == 0.0 and hidden.feasible
    late = solve_theta(64.0, dataclasses.replace(params, overhead_ms=20.0))
    assert late.theta == 1.0 and not late.feasible and abs(late.residual_ms - 10.0) <= 1e-9
    with pytest.raises(ValueError):
        solve_theta(-1.0, params)


def test_c06_dominance_and_calibration():
    rng = np.random.default_rng(66)
    for case in range(1000):
        n_layers = int(rng.integers(1, 10))
        loads = [LayerLoad(d_cold=float(rng.uniform(0, 40)) * (rng.random() < 0.6),
                           d_warm=float(rng.uniform(0, 150)) * (rng.random() < 0.9),
                           eval_ms=float(rng.uniform(0, 2)) * (rng.random() < 0.5)) for _ in range(n_layers)]
        params = PipelineParams(compute_ms=float(rng.uniform(0.5, 25)), overhead_ms=float(rng.uniform(0, 6)),
                                bw_hot_warm=float(rng.uniform(0.5, 32)), bw_warm_cold=float(rng.uniform(0.5, 8)),
                                compress_ratio=float(rng.uniform(0.05, 1.0)),
                                decompress_rate=float(rng.uniform(1, 64)))
        t = compare_modes(loads, params)
        assert t["dtp"] <= t["prefetch"] + 1e-9 and t["prefetch"] <= t["none"] + 1e-9, case
    sched = build_schedule([LayerLoad(d_warm=9.06) for _ in range(40)],
                           PipelineParams(compute_ms=3.125, overhead_ms=0.0, bw_hot_warm=1.0), "prefetch")
    for timing in sched.layers[1:]:
        assert abs(timing.idle_ms - 5.935) <= 1e-9
    serial = build_schedule([LayerLoad(d_warm=290.0, eval_ms=3.0)],
                            PipelineParams(compute_ms=100.0, overhead_ms=0.0, bw_hot_warm=1.0), "none")
    assert abs(serial.total_ms - 393.0) <= 1e-9
    lat = sched.layer_latencies()
    assert abs(sum(lat) - sched.total_ms) <= 1e-9


@pytest.mark.gpu
def test_host_tier_stream_and_split():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import oracle as O
    from paper_2506_20187_b200 import ops
    from paper_2506_20187_b200.tier import HostTier, kv_dequant
    lanes, n, d = 4, 4096, 128
    rng = np.random.default_rng(0)
    keys = torch.from_numpy(rng.normal(size=(lanes, n, d)).astype(np.float32)).to(torch.bfloat16)
    tier = HostTier(keys)
    dst = torch.zeros((lanes, n, d), dtype=torch.bfloat16, device="cuda")
    ranges = [(s, s + 64) for s in range(0, n, 256)]
    ev = tier.stream(dst, ranges, theta=0.5)
    torch.cuda.current_stream().wait_event(ev)
    got = dst.float().cpu().numpy()
    n_comp = (len(ranges) + 1) // 2
    kf = keys.float().numpy()
    for j, (s, e) in enumerate(ranges):
        if j < n_comp:  # INT4 path: dequantised records, rounded to bf16
            for i in range(lanes):
                ref = O.i4_dequant(O.i4_quant(kf[i, s:e]), d)
                ref = torch.from_numpy(ref).to(torch.bfloat16).float().numpy()
                assert np.array_equal(got[i, s:e], ref)
        else:
            assert np.array_equal(got[:, s:e], kf[:, s:e])
    untouched = np.ones(n, bool)
    for s, e in ranges:
        untouched[s:e] = False
    assert np.all(got[:, untouched] == 0)
    cal = tier.calibrate(dst)
    assert cal["bw_hot_warm"] > 0 and 0.3 < cal["compress_ratio"] < 0.32


def test_theta_for_rows_follows_solve_theta():
    """The DTP controller of host_tier (theta per layer from last step's promotions) is
    pipeline.py's solve_theta on the raw bf16 volume of those records."""
    from paper_2506_20187_b200.host_tier import theta_for_rows
    from paper_2506_20187_b200.tier import PipelineParams, solve_theta
    p = PipelineParams(compute_ms=0.5, bw_hot_warm=50e6, compress_ratio=80 / 256, decompress_rate=3e9)
    rows = [{"promotions": n} for n in (0, 100, 5000, 10 ** 6)]
    th = theta_for_rows(rows, p, 64, 128)
    assert th == [solve_theta(n * 64 * 128 * 2, p).theta for n in (0, 100, 5000, 10 ** 6)]
    assert th[0] == 0.0 and th[-1] == 1.0 and 0.0 <= th[2] <= 1.0
