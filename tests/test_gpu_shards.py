"""GPU parity of the vertex-partitioned G-shard schedule (DESIGN.md
"Multi-GPU") against the oracle's orc_train(G).

One B200 is available, so the multi-GPU semantics are checked three ways,
none of which has kernels on one GPU waiting on another process:
  * the dataflow epoch kernel running ALL G shards of the schedule in one
    launch (cfg.shards = G) -- the shard ordering, per-shard partitions,
    per-(step, shard) negatives, step-based windows and first-failure
    order the multi-GPU kernels execute;
  * a world-1 ShardedDevice: the IPC-attached path (replica control block,
    device barriers, failure/loss exchange) with no peers;
  * the per-step all-gather driver (dist.train_allgather) on the CUDA
    per-step operators over a world-1 process group.
Tolerances as in test_gpu_parity.py.
"""
import os
import socket

import numpy as np
import pytest

from test_gpu_parity import LOSS_RTOL, kind_model, z_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev(f2v):
    d = f2v.Device(0)
    yield d
    d.close()


def _graph(f2v, orc, n=1500, seed=3):
    rp, col = orc.orc_sbm_graph(n, 6, 0.03, 0.002, seed)
    return f2v.CsrGraph(rp, col)


@pytest.mark.parametrize("precision", ["fast", "exact"])
@pytest.mark.parametrize("G,kind,sampler,d,b", [
    (2, "sigmoid", "philox", 128, 64),
    (3, "tdist", "splitmix", 128, 50),
    (8, "tdist", "philox", 64, 32),
    (4, "sigmoid", "splitmix", 16, 40),
    (2, "fr", "philox", 2, 64),
])
def test_sharded_epochs_match_oracle(f2v, orc, dev, precision, G, kind, sampler, d, b):
    g = _graph(f2v, orc)
    n = g.num_vertices()
    z0 = np.zeros((n, d), np.float32)
    orc.oracle().orc_random_embedding(n, d, 3, z0)
    if kind == "fr":
        z0 *= 0.05
    mon = kind in ("sigmoid", "tdist")
    cfg = f2v.TrainConfig(dim=d, batch=b, negatives=5, lr=0.02, epochs=3,
                          model=kind_model(f2v, kind), seed=9, monitor_loss=mon,
                          sampler=sampler, precision=precision, shards=G)
    dev.upload_graph(g)
    dev.set_embedding(z0)
    ctr = f2v.TrainCounters()
    losses = dev.train_epochs(cfg, 0, 1, counters=ctr)
    z = dev.get_embedding()
    rc, zr, lr_, cr, _ = orc.orc_train(g.row_offsets, g.col_indices, z0, b, 5, 0.02, 1, kind, 9,
                                       monitor=mon, sampler=sampler, G=G, threads=8)
    assert rc == 0
    z_parity(z, zr)
    if mon:
        assert losses[0] == pytest.approx(lr_[0], rel=LOSS_RTOL[precision])
    assert [ctr.attractive_evals, ctr.repulsive_evals] == [int(cr[0]), int(cr[1])]


def test_sharded_trajectory_and_determinism(f2v, orc, dev):
    """Three epochs run independently on both sides; two device runs are
    bitwise identical (fixed-order partial combination, no float atomics)."""
    g = _graph(f2v, orc, 2500, 5)
    n = g.num_vertices()
    z0 = np.zeros((n, 128), np.float32)
    orc.oracle().orc_random_embedding(n, 128, 4, z0)
    cfg = f2v.TrainConfig(dim=128, batch=96, negatives=5, lr=0.02, epochs=3,
                          model=kind_model(f2v, "tdist"), seed=2, monitor_loss=True,
                          sampler="philox", shards=4, lr_decay="linear_to_zero")
    outs = []
    for _ in range(2):
        dev.upload_graph(g)
        dev.set_embedding(z0)
        outs.append((dev.train_epochs(cfg), dev.get_embedding()))
    assert outs[0][0] == outs[1][0] and np.array_equal(outs[0][1], outs[1][1])
    rc, zr, lr_, _, _ = orc.orc_train(g.row_offsets, g.col_indices, z0, 96, 5, 0.02, 3, "tdist",
                                      2, sampler="philox", G=4, lr_decay=True, threads=8)
    assert rc == 0
    np.testing.assert_allclose(outs[0][0], lr_, rtol=1e-3)
    rel = np.linalg.norm(outs[0][1].astype(np.float64) - zr) / np.linalg.norm(zr)
    assert rel < 1e-4, rel


def test_sharded_numerical_error_first_failure(f2v, orc, dev):
    rp, col = orc.orc_sbm_graph(300, 3, 0.1, 0.01, 5)
    g = f2v.CsrGraph(rp, col)
    z0 = np.zeros((300, 8), np.float32)
    orc.oracle().orc_random_embedding(300, 8, 2, z0)
    z0[123] = 3e37  # FR attraction r^2 overflows fp32 for 123's neighbours
    cfg = f2v.TrainConfig(dim=8, batch=16, negatives=3, lr=0.02, epochs=2,
                          model=kind_model(f2v, "fr"), seed=6, shards=3)
    dev.upload_graph(g)
    dev.set_embedding(z0)
    fail = {}
    with pytest.raises(f2v.NumericalError, match=r"non-finite gradient for vertex \d+ "
                                                 r"\(epoch 0, batch \d+\)"):
        dev.train_epochs(cfg, failure=fail)
    rc, zr, _, _, finfo = orc.orc_train(rp, col, z0, 16, 3, 0.02, 2, "fr", 6, monitor=False, G=3)
    assert rc == 4
    assert (fail["epoch"], fail["batch"], fail["vertex"]) == tuple(int(x) for x in finfo)
    z_parity(dev.get_embedding(), zr)


def test_world1_sharded_device_ipc_path(f2v, orc):
    """ShardedDevice with world 1: attach (own replicas), the per-epoch device
    barriers and the failure/loss exchange through the control block."""
    from paper_2009_10035_b200.dist import ShardedDevice

    g = _graph(f2v, orc, 1200, 7)
    n = g.num_vertices()
    z0 = np.zeros((n, 128), np.float32)
    orc.oracle().orc_random_embedding(n, 128, 6, z0)
    cfg = f2v.TrainConfig(dim=128, batch=128, negatives=5, lr=0.02, epochs=2,
                          model=kind_model(f2v, "sigmoid"), seed=3, monitor_loss=True,
                          sampler="philox")
    sd = ShardedDevice(rank=0, world=1, device=0)
    try:
        sd.setup(g, z0)
        losses = sd.train_epochs(cfg)
        z = sd.get_embedding()
        launches = sd.kernel_launches
    finally:
        sd.close()
    rc, zr, lr_, _, _ = orc.orc_train(g.row_offsets, g.col_indices, z0, 128, 5, 0.02, 2,
                                      "sigmoid", 3, sampler="philox", threads=8)
    assert rc == 0
    np.testing.assert_allclose(losses, lr_, rtol=1e-6)
    rel = np.linalg.norm(z.astype(np.float64) - zr, axis=1) / np.linalg.norm(zr, axis=1)
    assert rel.max() < 1e-5
    assert launches > 0


@pytest.mark.parametrize("backend", ["gloo", "nccl"])
def test_allgather_driver_on_device(f2v, orc, backend):
    """dist.train_allgather over the CUDA per-step operators (world-1 group;
    NCCL = the reference-granularity all-gather baseline on GPUs): per-step
    grad + failure vote + apply + row exchange."""
    import torch
    import torch.distributed as dist

    from paper_2009_10035_b200.dist import DeviceBackend, train_allgather

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if backend == "nccl":
        torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=0, world_size=1)
    tdev = torch.device("cuda", 0) if backend == "nccl" else None
    try:
        g = _graph(f2v, orc, 900, 2)
        n = g.num_vertices()
        z0 = np.zeros((n, 64), np.float32)
        orc.oracle().orc_random_embedding(n, 64, 8, z0)
        cfg = f2v.TrainConfig(dim=64, batch=64, negatives=5, lr=0.02, epochs=2,
                              model=kind_model(f2v, "tdist"), seed=5, monitor_loss=True,
                              sampler="philox")
        with f2v.Device(0) as dv:
            dv.upload_graph(g)
            dv.set_embedding(z0)
            losses = train_allgather(DeviceBackend(dv), g, cfg, 0, 1, tensor_device=tdev)
            z = dv.get_embedding()
            rows = dv.get_rows(np.array([3, 1, 3], np.uint32))
            assert np.array_equal(rows, z[[3, 1, 3]])
    finally:
        dist.destroy_process_group()
    rc, zr, lr_, _, _ = orc.orc_train(g.row_offsets, g.col_indices, z0, 64, 5, 0.02, 2, "tdist",
                                      5, sampler="philox", threads=8)
    assert rc == 0
    z_parity(z, zr)
    np.testing.assert_allclose(losses, lr_, rtol=1e-9)


@pytest.mark.parametrize("precision", ["fast", "exact"])
@pytest.mark.parametrize("G,kind,d", [(2, "sigmoid", 128), (3, "tdist", 128), (8, "tdist", 128),
                                      (4, "sigmoid", 128)])
def test_emulated_replicas_match_oracle(f2v, orc, dev, precision, G, kind, d):
    """The G-GPU data flow inside ONE launch (the safe stand-in for G GPUs on
    one device): shard g's items read and publish into their own Znew
    replica, and every finished row reaches the other replicas only through
    the peer-store epilogue (store_peers) -- so readers poll sentinels of
    rows written by "peers".  After every epoch all replicas are checked equal
    on the device; Z must equal orc_train(G) and the one-replica run bit for
    bit."""
    g = f2v.rmat_graph(12, 16, seed=G)  # skewed degrees: uneven work-balanced shards
    n = g.num_vertices()
    z0 = np.zeros((n, d), np.float32)
    orc.oracle().orc_random_embedding(n, d, 5, z0)
    cfg = f2v.TrainConfig(dim=d, batch=48, negatives=5, lr=0.02, epochs=2,
                          model=kind_model(f2v, kind), seed=3, monitor_loss=True,
                          sampler="philox", precision=precision, shards=G)
    outs = []
    for emul in (False, True):
        if emul:
            os.environ["F2V_EMULATE_REPLICAS"] = "1"
        try:
            dev.upload_graph(g)
            dev.set_embedding(z0)
            losses = dev.train_epochs(cfg)
            outs.append((losses, dev.get_embedding()))
        finally:
            os.environ.pop("F2V_EMULATE_REPLICAS", None)
    assert outs[0][0] == outs[1][0] and np.array_equal(outs[0][1], outs[1][1])
    rc, zr, lr_, _, _ = orc.orc_train(g.row_offsets, g.col_indices, z0, 48, 5, 0.02, 2, kind, 3,
                                      sampler="philox", G=G, threads=8)
    assert rc == 0
    np.testing.assert_allclose(outs[1][0], lr_, rtol=1e-3)
    rel = np.linalg.norm(outs[1][1].astype(np.float64) - zr) / np.linalg.norm(zr)
    assert rel < 1e-4, rel


@pytest.mark.parametrize("precision,sampler,kind", [("exact", "splitmix", "sigmoid"),
                                                    ("exact", "philox", "tdist"),
                                                    ("fast", "philox", "sigmoid"),
                                                    ("fast", "philox", "tdist")])
def test_nccl_allgather_library_world1(f2v, orc, precision, sampler, kind):
    """The in-library per-step ncclAllGather baseline (f2v_train_epochs_allgather,
    world-1 NCCL communicator): device-resident grad -> pack -> all-gather ->
    vote -> scatter per step, no host staging.  Against the oracle's train();
    EXACT with the reference's own streams is bit-identical in practice."""
    from paper_2009_10035_b200.dist import AllgatherDevice

    g = _graph(f2v, orc, 1800, 4)
    n = g.num_vertices()
    z0 = np.zeros((n, 128), np.float32)
    orc.oracle().orc_random_embedding(n, 128, 2, z0)
    cfg = f2v.TrainConfig(dim=128, batch=100, negatives=5, lr=0.02, epochs=2,
                          model=kind_model(f2v, kind), seed=4, monitor_loss=True,
                          sampler=sampler, precision=precision)
    ag = AllgatherDevice(rank=0, world=1, device=0)
    try:
        ag.setup(g, z0)
        ctr = f2v.TrainCounters()
        losses = ag.train_epochs(cfg, counters=ctr)
        z = ag.get_embedding()
    finally:
        ag.close()
    rc, zr, lr_, cr, _ = orc.orc_train(g.row_offsets, g.col_indices, z0, 100, 5, 0.02, 2, kind,
                                       4, sampler=sampler, threads=8)
    assert rc == 0
    _, _, same = z_parity(z, zr)
    if precision == "exact":
        assert same >= 0.9999, same
    np.testing.assert_allclose(losses, lr_, rtol=LOSS_RTOL[precision])
    assert [ctr.attractive_evals, ctr.repulsive_evals] == [int(cr[0]), int(cr[1])]


def test_nccl_allgather_library_failure(f2v, orc):
    """A non-finite gradient stops every rank at the oracle's (epoch, batch,
    vertex), Z left at the last complete step (trainer.cpp:149-152)."""
    from paper_2009_10035_b200.dist import AllgatherDevice

    rp, col = orc.orc_sbm_graph(300, 3, 0.1, 0.01, 5)
    g = f2v.CsrGraph(rp, col)
    z0 = np.zeros((300, 128), np.float32)
    orc.oracle().orc_random_embedding(300, 128, 2, z0)
    z0[123] = 3e37  # FR attraction r^2 overflows fp32 for 123's neighbours
    cfg = f2v.TrainConfig(dim=128, batch=16, negatives=3, lr=0.02, epochs=2,
                          model=kind_model(f2v, "fr"), seed=6, precision="exact")
    ag = AllgatherDevice(rank=0, world=1, device=0)
    fail = {}
    try:
        ag.setup(g, z0)
        with pytest.raises(f2v.NumericalError, match=r"non-finite gradient for vertex \d+ "
                                                     r"\(epoch 0, batch \d+\)"):
            ag.train_epochs(cfg, failure=fail)
        z = ag.get_embedding()
    finally:
        ag.close()
    rc, zr, _, _, finfo = orc.orc_train(rp, col, z0, 16, 3, 0.02, 2, "fr", 6, monitor=False)
    assert rc == 4
    assert (fail["epoch"], fail["batch"], fail["vertex"]) == tuple(int(x) for x in finfo)
    z_parity(z, zr)


def test_nccl_before_torch_import():
    """The library's NCCL (run-time dlopen) must not shadow torch's bundled
    NCCL: creating the per-step baseline's communicator before `import torch`
    left torch unable to resolve its newer NCCL symbols (round-2 bench)."""
    import subprocess
    import sys

    from conftest import ROOT
    code = ("import sys; sys.path.insert(0, %r); import paper_2009_10035_b200 as f2v; "
            "uid = f2v.Device.nccl_unique_id(); import torch; "
            "print('OK', len(uid), torch.cuda.is_available())" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().startswith("OK 128"), out.stdout
