"""GPU parity of the HELR deployer (NEXT f3, uellm_helr_plan) against the oracle (O12): the
chosen chain, layer ranges, mask and both doubles bit-identical (same explicitly rounded
operations in the same order)."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu


def gpu_helr(t, device_out=False):
    from paper_2409_14961_b200 import uellm as U
    D = len(t.memory_bytes)
    wsb = U.helr_workspace_bytes(D)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda:0")
    if not device_out:
        return U.helr_plan(t, ws, wsb).as_dict()
    out = torch.zeros(U.C.sizeof(U.DeviceMap), dtype=torch.uint8, device="cuda:0")
    U.helr_plan(t, ws, wsb, out)
    torch.cuda.synchronize()
    return U.DeviceMap.from_buffer_copy(out.cpu().numpy().tobytes()).as_dict()


@pytest.mark.parametrize("seed", range(60))
def test_helr_small_random(seed):
    t = W.random_topology(seed, 1 + seed % 8)
    assert gpu_helr(t) == oracle.helr(t)


@pytest.mark.parametrize("nodes,per_node", [(1, 8), (2, 8), (1, 4)])
@pytest.mark.parametrize("a", [(1.0, 1.0), (0.0, 1.0), (10.0, 1.0)])
def test_helr_b200_clusters(nodes, per_node, a):
    t = W.b200_cluster(nodes=nodes, per_node=per_node, seed=nodes * 10 + per_node).replace(a1=a[0], a2=a[1])
    g = gpu_helr(t, device_out=True)
    assert g == oracle.helr(t)
    assert g["feasible"] and sum(g["layer_count"]) == t.num_layers


def test_helr_max_devices():
    t = W.b200_cluster(nodes=3, per_node=8, seed=3)
    t = t.replace(memory_bytes=t.memory_bytes[:20], performance=t.performance[:20],
                  link_latency_s=np.ascontiguousarray(t.link_latency_s[:20, :20]))
    assert gpu_helr(t) == oracle.helr(t)


def test_helr_infeasible_and_config_errors():
    from paper_2409_14961_b200 import uellm as U
    t = W.Topology(np.array([10, 10], np.uint64), np.array([1.0, 1.0]), np.zeros((2, 2)), num_layers=8,
                   model_bytes=1000)
    g = gpu_helr(t)
    assert g == oracle.helr(t) and not g["feasible"]
    ws = torch.empty(U.helr_workspace_bytes(2), dtype=torch.uint8, device="cuda:0")
    for bad in (t.replace(performance=np.array([1.0, 0.0])), t.replace(a1=-1.0),
                t.replace(link_latency_s=np.array([[0, np.nan], [np.nan, 0]]))):
        with pytest.raises(U.UellmError) as e:
            U.helr_plan(bad, ws, ws.numel())
        assert e.value.status == U.ERR_CONFIG


def gpu_bgs(t):
    from paper_2409_14961_b200 import uellm as U
    D = len(t.memory_bytes)
    wsb = U.helr_workspace_bytes(D)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda:0")
    return U.bgs_plan(t, ws, wsb).as_dict()


@pytest.mark.parametrize("seed", range(40))
def test_bgs_small_random(seed):
    t = W.random_topology(seed, 1 + seed % 8)
    assert gpu_bgs(t) == oracle.bgs(t)


def test_bgs_b200_cluster_vs_helr():
    t = W.b200_cluster(nodes=2, per_node=8, seed=5)
    b = gpu_bgs(t)
    assert b == oracle.bgs(t)
    assert gpu_helr(t)["objective"] <= b["objective"]
