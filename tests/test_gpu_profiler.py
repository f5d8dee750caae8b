"""GPU parity of the profiler stand-ins + misprediction monitor (NEXT f4, uellm_predict_lengths)
against the oracle (O9-O11): predicted lengths, per-window inflation factors and the correction
count bit-exact; and the predictions feeding the scheduling path end to end."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu
P = W.PredictorConfig


def gpu_predict(t, pc, factor0=1.0, levels=True):
    from paper_2409_14961_b200 import uellm as U
    dev = torch.device("cuda:0")
    n = len(t)
    st = U.MonitorState()
    st.inflation_factor = factor0
    d_state = torch.frombuffer(bytearray(bytes(st)), dtype=torch.uint8).to(dev)
    d_t = torch.from_numpy(np.ascontiguousarray(t, np.uint32).view(np.int32)).to(dev)
    d_p = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
    wl = pc.window or max(n, 1)
    nwin = (n + wl - 1) // wl
    d_f = torch.zeros(nwin + 1, dtype=torch.float64, device=dev)
    cp = U.make_predictor(pc)
    wsb = U.predict_workspace_bytes(n, cp) if levels else 0
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    U.predict_lengths(n, d_t if n else None, cp, d_state, d_p if n else None, d_f, ws=ws if wsb else None,
                      ws_bytes=wsb)
    torch.cuda.synchronize()
    s = U.MonitorState.from_buffer_copy(d_state.cpu().numpy().tobytes())
    return d_p[:n].cpu().numpy().view(np.uint32), d_f.cpu().numpy(), s


@pytest.mark.parametrize("pc", [P(variant=0, window=1000), P(variant=1, bucket_width=16, window=777),
                                P(variant=2, error_rate=0.0049, bucket_width=16, window=5000, seed=3),
                                P(variant=2, error_rate=0.4, bucket_width=32, window=999, seed=4),
                                P(variant=2, error_rate=1.0, bucket_width=8, window=0, seed=5),
                                P(variant=3, constant_tokens=64, window=2048, gamma=1.01, cap=3.0),
                                P(variant=3, constant_tokens=1, window=100, monitor=0)])
@pytest.mark.parametrize("levels", [True, False])
def test_predict_parity(pc, levels):
    t = W.true_output_lengths(60_000, 7)
    pred, factors, st = gpu_predict(t, pc, levels=levels)
    o_pred, o_factors, o_corr = oracle.profile_stream(t, pc)
    assert np.array_equal(pred, o_pred)
    assert np.array_equal(factors, o_factors)            # bit-identical doubles (same operation order)
    assert st.corrections == o_corr and st.inflation_factor == o_factors[-1]
    assert list(st.scratch) == [0, 0]


@pytest.mark.parametrize("levels", [True, False])
def test_predict_factor0_and_saturation(levels):
    t = np.full(5000, 4_000_000_000, np.uint32)
    pc = P(variant=0, window=1000)
    pred, factors, st = gpu_predict(t, pc, factor0=1.5, levels=levels)
    o_pred, o_factors, o_corr = oracle.profile_stream(t, pc, factor0=1.5)
    assert np.array_equal(pred, o_pred) and np.all(pred == 2**32 - 1)
    assert np.array_equal(factors, o_factors) and st.corrections == o_corr


def test_predict_level_path_applicability():
    from paper_2409_14961_b200 import uellm as U
    assert U.predict_workspace_bytes(10**6, U.make_predictor(P(window=1000))) > 0
    assert U.predict_workspace_bytes(10**6, U.make_predictor(P(window=1000, gamma=1.0001))) == 0   # too many levels
    assert U.predict_workspace_bytes(10**6, U.make_predictor(P(window=1000, monitor=0, gamma=1.0001))) > 0


def test_predict_many_levels_window_path():
    t = W.true_output_lengths(30_000, 9)
    pc = P(variant=3, constant_tokens=20, window=300, gamma=1.001, cap=4.0)
    pred, factors, st = gpu_predict(t, pc)          # no level workspace available: window path
    o_pred, o_factors, o_corr = oracle.profile_stream(t, pc)
    assert np.array_equal(pred, o_pred) and np.array_equal(factors, o_factors) and st.corrections == o_corr


@pytest.mark.parametrize("levels", [True, False])
def test_predict_full_size_stream(levels):
    """c4's shape: 10^8 true lengths, one monitor epoch per 10^6-query window."""
    t = W.true_output_lengths(100_000_000, 0)
    pc = P(variant=2, error_rate=0.0049, bucket_width=16, window=1_000_000, seed=0)
    pred, factors, st = gpu_predict(t, pc, levels=levels)
    o_pred, o_factors, o_corr = oracle.profile_stream(t, pc)
    assert np.array_equal(pred, o_pred) and np.array_equal(factors, o_factors) and st.corrections == o_corr


def test_predictions_feed_the_schedule():
    """f4 -> a1..a8: the GPU's predicted lengths scheduled on the GPU equal the oracle chain."""
    from paper_2409_14961_b200.scheduler import GpuScheduler
    n = 200_000
    inp, _, slo = W.long_tail(n, 3)
    t = W.true_output_lengths(n, 3)
    pc = P(variant=2, error_rate=0.05, bucket_width=16, window=50_000, seed=1)
    pred, _, _ = gpu_predict(t, pc)
    cfg = W.c3(0, n=10)[3].replace(window=50_000)
    g = GpuScheduler(n, cfg, device="cuda:0")
    g.run(torch.from_numpy(inp.view(np.int32)).cuda(), torch.from_numpy(pred.view(np.int32)).cuda(),
          torch.from_numpy(slo).cuda())
    r = g.results()
    o_pred, _, _ = oracle.profile_stream(t, pc)
    o_order, o_offs, o_m, o_cost = oracle.schedule(inp, o_pred, slo, cfg, nthreads=8)
    assert np.array_equal(r["order"], o_order) and np.array_equal(r["offsets"], o_offs)
    assert r["totals"]["dp_cost"] == o_cost


def test_predict_empty_and_config_errors():
    from paper_2409_14961_b200 import uellm as U
    pred, factors, st = gpu_predict(np.zeros(0, np.uint32), P(variant=1), factor0=1.25)
    assert factors[0] == 1.25 and st.corrections == 0
    t = torch.ones(10, dtype=torch.int32, device="cuda:0")
    p = torch.zeros(10, dtype=torch.int32, device="cuda:0")
    s = torch.zeros(32, dtype=torch.uint8, device="cuda:0")
    for bad in (P(variant=4), P(variant=1, bucket_width=0), P(variant=3, constant_tokens=0),
                P(error_rate=1.5), P(gamma=0.5), P(monitor=2)):
        with pytest.raises(U.UellmError) as e:
            U.predict_lengths(10, t, U.make_predictor(bad), s, p)
        assert e.value.status == U.ERR_CONFIG
    with pytest.raises(U.UellmError) as e:          # host state pointer
        U.predict_lengths(10, t, U.make_predictor(P()), C.addressof(U.MonitorState()), p)
    assert e.value.status == U.ERR_ARG
