"""Multi-GPU host logic on CPU (no GPU): the vertex-partitioned G-shard
schedule run as real
world_size-2 / 3 process groups over gloo.

* shard layout / per-shard Fisher-Yates / shard negatives of the host library
  against the oracle;
* paper_2009_10035_b200.dist.train_allgather -- the per-step all-gather
  driver the NCCL baseline uses -- with the oracle as each rank's compute
  backend (test infrastructure), against orc_train(G): Z bit-identical, loss
  trajectory identical, a non-finite gradient raised on every rank with the
  oracle's (epoch, batch, vertex) and Z left at the last complete step;
* the IPC-handle all-gather of ShardedDevice.setup.
"""
import os
import socket
import sys

import numpy as np
import pytest

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


GAMMA = 0x9e3779b97f4a7c15
M64 = (1 << 64) - 1


def _mix(z):  # rng.hpp:44-49
    z = (z + GAMMA) & M64
    z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & M64
    z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & M64
    return z ^ (z >> 31)


def test_shard_layout_matches_oracle(f2v, orc):
    """The product's shard layout equals the oracle's definition
    (orc_shard_layout): work-quantile row bounds, per-shard batches, and the
    combined step-major positions."""
    graphs = [f2v.rmat_graph(12, 16, seed=2), f2v.sbm_graph(1001, 7, 0.02, 0.002, 3),
              f2v.CsrGraph(np.zeros(38, np.uint64), np.zeros(0, np.uint32)),
              f2v.CsrGraph(np.zeros(11, np.uint64), np.zeros(0, np.uint32))]
    for g in graphs:
        n = g.num_vertices()
        for b, G, s in [(64, 2, 5), (64, 3, 5), (8, 8, 1), (64, 3, 6), (256, 1, 5)]:
            if n < G:
                continue
            lo, bs, poff, T = f2v.shard_layout(g, b, G, s)
            rlo, rbs, rnb, rT = orc.orc_shard_layout(g.row_offsets, G, s, b)
            assert np.array_equal(lo, rlo) and np.array_equal(bs, rbs) and T == rT
            assert lo[0] == 0 and lo[G] == n and np.all(np.diff(lo.astype(np.int64)) >= 1)
            pos = 0
            for t in range(T):
                for k in range(G):
                    assert poff[t * G + k] == pos
                    if t < rnb[k]:
                        pos += min(int(bs[k]), int(lo[k + 1] - lo[k]) - t * int(bs[k]))
            assert poff[T * G] == pos == n
    with pytest.raises(f2v.UsageError):
        f2v.shard_layout(f2v.CsrGraph(np.zeros(4, np.uint64), np.zeros(0, np.uint32)), 4, 4, 5)


def test_shard_layout_balances_rmat_work(f2v, orc):
    """R-MAT's hub rows have low ids: equal row ranges gave shard 0 of 8
    ~42% of the arcs.  Work-quantile bounds keep every shard
    within a few percent of 1/G of the work, and every shard's step count
    within one of T."""
    g = f2v.rmat_graph(16, 16, seed=1)
    n, s = g.num_vertices(), 5
    w = g.degrees() + s
    for G in (2, 4, 8):
        lo, bs, poff, T = f2v.shard_layout(g, 384, G, s)
        share = np.array([w[lo[k]:lo[k + 1]].sum() for k in range(G)]) / w.sum()
        assert share.max() <= 1.0 / G + 0.01, share
        nb = [-(-int(lo[k + 1] - lo[k]) // int(bs[k])) for k in range(G)]
        assert max(nb) == T and min(nb) >= T - 1, (nb, T)


def test_partition_shard_matches_oracle(f2v, orc):
    for (n, b, seed, epoch, g, G) in [(500, 32, 7, 0, 0, 1), (333, 16, 7, 3, 1, 2),
                                      (250, 250, 1, 2, 2, 3)]:
        key = [0x22, epoch] if G == 1 else [0x22, epoch, g]
        ref = orc.orc_partition(n, b, orc.orc_rng_keyed(seed, key))
        assert np.array_equal(f2v.partition_shard(n, b, seed, epoch, g, G), ref)
    # G == 1 is train()'s own partition_epoch
    assert np.array_equal(f2v.partition_shard(500, 32, 3, 1, 0, 1), f2v.partition_epoch(500, 32, 3, 1))


def test_shard_negatives_match_oracle(f2v, orc):
    for sampler in ("philox", "splitmix"):
        for g, G in [(0, 1), (1, 2), (2, 3)]:
            ours = f2v.negatives(sampler, 5, 1, 7, 1000, 5, shard=g, num_shards=G)
            if sampler == "philox":
                ref = orc.orc_negatives("philox", 5, 1, 7, 1000, 5, gpu=g)
            elif G == 1:
                ref = orc.orc_negatives("splitmix", 5, 1, 7, 1000, 5)
            else:  # draw k of Rng::keyed(seed,{0x33,epoch,batch,shard}) (rng.hpp:26-42)
                st = orc.orc_rng_keyed(5, [0x33, 1, 7, g])
                ref = np.array([(_mix(st + (k + 1) * GAMMA) * 1000) >> 64 for k in range(5)],
                               np.uint32)
            assert np.array_equal(ours, ref), (sampler, g, G)


# ----------------------------------------------------------- gloo workers
def _worker(rank, world, port, case, q):
    try:
        sys.path.insert(0, ROOT)
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist

        import paper_2009_10035_b200 as f2v
        import pyoracle as orc
        from paper_2009_10035_b200 import dist as f2vdist

        dist.init_process_group("gloo", rank=rank, world_size=world)

        class OracleBackend(f2vdist.StepBackend):
            """test infrastructure: the oracle as one rank's compute"""

            def __init__(self, g, z):
                self.rp, self.col, self.z, self.d = g.row_offsets, g.col_indices, z, z.shape[1]

            def grad(self, ids, negs, cfg):
                rc, gr, bad = orc.orc_grad_minibatch(self.rp, self.col, self.z, ids, negs,
                                                     "sigmoid" if int(cfg.model.kind) == 0
                                                     else "tdist")
                if rc:
                    raise f2v.NumericalError(f"non-finite gradient for vertex {bad}")
                return gr

            def loss(self, ids, negs, cfg):
                return orc.orc_batch_loss(self.rp, self.col, self.z, ids, negs,
                                          "sigmoid" if int(cfg.model.kind) == 0 else "tdist")

            def apply(self, ids, grads, eta):  # trainer.cpp:167-175, fp32 mul then sub
                for i, u in enumerate(ids):
                    self.z[u] = self.z[u] - np.float32(eta) * grads[i]

            def get_rows(self, ids):
                return self.z[ids].copy()

            def set_rows(self, ids, rows):
                self.z[ids] = rows

        g = f2v.sbm_graph(case["n"], 4, 0.08, 0.01, 3)
        z = case["z0"].copy()
        be = OracleBackend(g, z)
        cfg = f2v.TrainConfig(dim=z.shape[1], batch=case["b"], negatives=5, lr=0.02,
                              epochs=case["epochs"], model=f2v.ForceModel(case["kind"]), seed=11,
                              monitor_loss=True, sampler=case["sampler"],
                              lr_decay=case.get("decay", "constant"))
        err = None
        try:
            losses = f2vdist.train_allgather(be, g, cfg, rank, world)
        except f2v.NumericalError as e:
            losses, err = None, str(e)
        # the IPC-handle exchange of ShardedDevice.setup (bytes objects)
        hs = f2vdist._all_gather_objects(bytes([rank]) * 192)
        q.put((rank, z, losses, err, [h[:1] for h in hs]))
        dist.destroy_process_group()
    except BaseException as e:  # surface worker failures
        import traceback
        q.put((rank, None, None, "WORKER " + traceback.format_exc(), None))


def _run(world, case):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r = q.get(timeout=300)
        out[r[0]] = r[1:]
    for p in procs:
        p.join(60)
    for r, v in out.items():
        assert v[2] is None or not v[2].startswith("WORKER"), v[2]
    return out


CASES = [
    dict(n=301, b=32, epochs=2, kind=0, sampler="philox"),
    dict(n=256, b=40, epochs=2, kind=1, sampler="splitmix", decay="linear_to_zero"),
]


@pytest.mark.parametrize("world,case", [(2, CASES[0]), (2, CASES[1]), (3, CASES[0])])
def test_allgather_schedule_matches_oracle_gloo(f2v, orc, world, case):
    rng = np.random.default_rng(5)
    case = dict(case, z0=rng.uniform(-1, 1, (case["n"], 16)).astype(np.float32))
    out = _run(world, case)
    g = f2v.sbm_graph(case["n"], 4, 0.08, 0.01, 3)
    rc, zr, lr_, _, _ = orc.orc_train(g.row_offsets, g.col_indices, case["z0"], case["b"], 5,
                                      0.02, case["epochs"], "sigmoid" if case["kind"] == 0 else
                                      "tdist", 11, sampler=case["sampler"], G=world,
                                      lr_decay=case.get("decay") == "linear_to_zero")
    assert rc == 0
    for r in range(world):
        z, losses, err, hs = out[r]
        assert err is None, err
        # every replica equals the oracle's G-shard Z, bit for bit
        assert np.array_equal(z, zr), (r, np.abs(z - zr).max())
        assert np.array_equal(np.array(losses), lr_), (losses, lr_)
        assert hs == [bytes([k]) for k in range(world)]


def test_allgather_failure_vote_matches_oracle_gloo(f2v, orc):
    n, d = 200, 8
    g = f2v.sbm_graph(n, 4, 0.08, 0.01, 3)
    z0 = np.random.default_rng(2).uniform(-1, 1, (n, d)).astype(np.float32)
    # two huge rows with a common neighbour: its sigmoid attraction overflows fp32
    deg = g.degrees()
    u = int(np.argmax(deg))
    v1, v2 = g.neighbors(u)[:2]
    z0[v1] = 3e38
    z0[v2] = 3e38
    z0[u] = -1.0
    case = dict(n=n, b=16, epochs=1, kind=0, sampler="philox", z0=z0)
    rc, zr, _, _, fail = orc.orc_train(g.row_offsets, g.col_indices, z0, 16, 5, 0.02, 1,
                                       "sigmoid", 11, sampler="philox", G=2)
    assert rc == 4
    out = _run(2, case)
    for r in range(2):
        z, losses, err, _ = out[r]
        assert err == f"non-finite gradient for vertex {fail[2]} (epoch {fail[0]}, batch {fail[1]})"
        assert np.array_equal(z, zr)
