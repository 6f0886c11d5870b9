#!/usr/bin/env python3
"""bench.py -- Force2Vec minibatch-SGD epochs on B200 (BASELINE.json metric:
edge+neg-sample updates/s and sec/epoch at d=128; % of HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config c3|c1|c2|c4|c5] [--precision exact|fast]

A "step" is one epoch of train() (trainer.cpp:211-249) over the whole graph:
every batch's fused gradient + update.  Default workload = BASELINE config 3,
the config north_star's target names (Chung-Lu n=3M power-law graph, 230M
directed arcs, sigmoid, d=128, b=384, s=5, lr=.02, Philox negatives,
Z ~ U(-1,1)), synthetic (no dataset), at the reference's arithmetic
(precision="exact": fp64 pair math and accumulation in the reference's order).

Printed JSON (rank 0, one line):
  value  = (nnz + n*s) * K / (device time of K epochs), inputs resident in HBM,
           timed with CUDA events on the library's stream;
  fast   = the same K epochs with precision="fast" (fp32 pair math, fp64
           accumulation) -- reported beside the headline, not as it;
  e2e    = same metric through the public API with host buffers: per step one
           full train() of the config's epoch schedule including H2D of CSR + Z
           from pinned memory and D2H of Z;
  roofline = algorithmic bytes per epoch-kernel launch / its event-timed
           duration vs MEASURED_PEAKS.json hbm_gbs; traffic from the committed
           ncu capture (profiles/ncu_traffic.json) of the same config+precision;
  cpu_baseline = the unmodified reference (oracle/_ref) on this host's cores
           over a bounded sample of batches.

--impl reference never loads the product library: the oracle's restated
generator emits the edge list, the reference's own from_edges builds the CSR
(once per process), and the reference core times a bounded sample of epoch 0
with the same Philox negatives the device draws.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

CONFIGS = {
    # name: (generator, kwargs, kind, d, b, s, lr, epochs)
    "c1": ("sbm", dict(n=4096, blocks=8, p_in=0.03, p_out=0.001, seed=4096), "sigmoid", 128, 256,
           5, 0.02, 10),
    "c2": ("rmat", dict(scale=20, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1), "tdist", 128,
           384, 5, 0.02, 5),
    "c3": ("chung_lu", dict(n=3_000_000, exponent=2.2, min_deg=2.0, max_deg=30000.0,
                            mean_deg=78.0, seed=1), "sigmoid", 128, 384, 5, 0.02, 1),
    "c4": ("rgg", dict(n=1_000_000, mean_deg=12.0, seed=1), "tdist", 2, 256, 5, 0.02, 20),
    "c5": ("rmat", dict(scale=26, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1), "sigmoid", 128,
           512, 5, 0.02, 1),
}
WORKLOAD_NAMES = {
    "c1": "SBM n=4096 (8 blocks, p_in .03, p_out .001), sigmoid, d=128, b=256, s=5, lr .02",
    "c2": "R-MAT scale 20 (ef 16, .57/.19/.19/.05), t-dist, d=128, b=384, s=5, lr .02",
    "c3": "Chung-Lu n=3M power-law 2.2 (min 2, max 30000, mean 78), sigmoid, d=128, b=384, s=5",
    "c4": "RGG n=1M unit square (mean degree 12), t-dist, d=2, b=256, s=5, lr .02",
    "c5": "R-MAT scale 26 (ef 16, .57/.19/.19/.05), sigmoid, d=128, b=512, s=5, lr .02",
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def make_graph(f2v, cfg_name):
    gen, kw, *_ = CONFIGS[cfg_name]
    t0 = time.perf_counter()
    if gen == "sbm":
        g = f2v.sbm_graph(kw["n"], kw["blocks"], kw["p_in"], kw["p_out"], kw["seed"])
    elif gen == "rmat":
        g = f2v.rmat_graph(kw["scale"], kw["edge_factor"], kw["a"], kw["b"], kw["c"], kw["seed"])
    elif gen == "chung_lu":
        g = f2v.chung_lu_graph(kw["n"], kw["exponent"], kw["min_deg"], kw["max_deg"],
                               kw["mean_deg"], kw["seed"])
    else:
        g = f2v.rgg_graph(kw["n"], kw["mean_deg"], kw["seed"])
    log(f"graph {cfg_name}: n={g.num_vertices()} nnz={g.num_edges()} "
        f"max_deg={int(g.degrees().max())} built in {time.perf_counter() - t0:.1f}s")
    return g


def algorithmic_bytes(n, nnz, d, b, s):
    """nnz(4d+4) + n(8d+20) + ceil(n/b) s (4d+4) bytes per epoch."""
    return nnz * (4 * d + 4) + n * (8 * d + 20) + ((n + b - 1) // b) * s * (4 * d + 4)


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.samples = []
        self.source = "nvidia-smi"
        self.nvml = None
        try:  # initialised before the timed region starts
            import pynvml as N
            N.nvmlInit()
            self.nvml = (N, N.nvmlDeviceGetHandleByIndex(device))
        except Exception:
            self.nvml = None
        self.stop = threading.Event()
        self.th = threading.Thread(target=self.run, daemon=True)

    def run(self):
        # NVML (microsecond queries, sampled every 5 ms) when available, so a
        # short timed region still gets many samples; nvidia-smi otherwise
        try:
            N, h = self.nvml
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            bits = [N.nvmlClocksThrottleReasonHwSlowdown,
                    N.nvmlClocksThrottleReasonHwThermalSlowdown,
                    N.nvmlClocksThrottleReasonSwThermalSlowdown,
                    N.nvmlClocksThrottleReasonSwPowerCap]
            while True:  # at least one sample, however short the timed region
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append([str(sm), str(mx)] +
                                    ["Active" if r & b else "Not Active" for b in bits])
                if self.stop.wait(0.002):
                    break
            self.source = "nvml"
            return
        except Exception:
            pass
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.1)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples), "source": self.source}


def ncu_traffic(cfg_name):
    """dram bytes per epoch-kernel launch from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
        e = t.get(cfg_name)
        return e["dram_bytes_per_launch"] if e else None
    except Exception:
        return None


def philox_negs(n, b, s, nb, epoch=0, seed=1):
    """The configs' Philox negatives of batches 0..nb-1 of one epoch (the same
    stream the device samples), from the oracle's restatement."""
    import pyoracle as P
    out = np.zeros(nb * s, np.uint32)
    for bi in range(nb):
        out[bi * s:(bi + 1) * s] = P.orc_negatives("philox", seed, epoch, bi, n, s)
    return out


def reference_graph(cfg_name):
    """The config's graph built without the product library: the oracle's
    restated generator (oracle/f2v_oracle_gen.c) emits the edge list, the
    reference's own CsrGraph::from_edges (csr_graph.cpp:57-97, oracle/_ref)
    builds the CSR.  Returns ("reference", RefGraph, n, nnz), or ("port",
    (rowptr, col), n, nnz) with the C restatement when _ref is absent."""
    import pyoracle as P
    gen, kw, *_ = CONFIGS[cfg_name]
    t0 = time.perf_counter()
    pairs, n = P.orc_gen_pairs(gen, **kw)
    t1 = time.perf_counter()
    if P.reference_available():
        rg = P.ref_graph_from_edges(pairs, n, True)
        del pairs
        nnz = P.reference().ref_graph_nnz(rg.ptr)
        log(f"graph {cfg_name} (oracle edge list {t1 - t0:.1f}s, reference from_edges "
            f"{time.perf_counter() - t1:.1f}s): n={n} nnz={nnz}")
        return "reference", rg, n, nnz
    rowptr, col, _, _ = P.orc_from_edges(pairs, n, True)
    log(f"graph {cfg_name} (oracle edge list + C restatement of from_edges "
        f"{time.perf_counter() - t0:.1f}s): n={n} nnz={len(col)}")
    return "port", (rowptr, col), n, len(col)


class ReferenceCPU:
    """The reference's CPU path on this host's cores over a bounded prefix of
    epoch 0's batches: partition_epoch + build_minibatch (Philox negatives
    injected, as the device draws them) + make_schedule + grad_minibatch +
    apply_update (trainer.cpp:210-236), monitoring off.  kind "reference" =
    the unmodified reference core (oracle/_ref); "port" = the C restatement."""

    def __init__(self, kind, graph, n, z0, cfg_name, workers=None):
        import pyoracle as P
        _, _, fkind, d, b, s, lr, _ = CONFIGS[cfg_name]
        self.P, self.kind, self.graph, self.n, self.z0 = P, kind, graph, n, z0
        self.fkind, self.d, self.b, self.s, self.lr = fkind, d, min(b, n), s, lr
        self.workers = workers or os.cpu_count()
        self.nb_total = (n + self.b - 1) // self.b
        self.negs = philox_negs(n, self.b, s, self.nb_total)
        if kind == "port":
            self.perm = P.orc_epoch_perm(n, self.b, 1, 0)

    def run(self, nb):
        import ctypes as C
        P = self.P
        z = np.array(self.z0, copy=True)
        if self.kind == "reference":
            pairs = C.c_uint64()
            secs = P.reference().ref_time_batches(
                self.graph.ptr, z, self.d, self.b, self.s, np.float32(self.lr),
                P.KINDS[self.fkind], 1, self.workers, nb, self.negs.ctypes.data_as(C.c_void_p),
                C.byref(pairs))
            return secs, pairs.value
        rowptr, col = self.graph
        t0 = time.perf_counter()
        pairs = 0
        for bi in range(nb):
            ids = self.perm[bi * self.b:(bi + 1) * self.b]
            negs = self.negs[bi * self.s:(bi + 1) * self.s]
            rc, grads, _ = P.orc_grad_minibatch(rowptr, col, z, ids, negs, self.fkind,
                                                threads=self.workers)
            P.oracle().orc_apply_update(z, self.d, ids, len(ids), grads, np.float32(self.lr))
            pairs += int((rowptr[ids + 1] - rowptr[ids]).sum()) + len(ids) * self.s
        return time.perf_counter() - t0, pairs

    def size_for(self, budget_s):
        probe = min(self.nb_total, 16)
        secs, _ = self.run(probe)
        return int(min(self.nb_total, max(probe, probe * budget_s / max(secs, 1e-6))))

    def measure(self, nb):
        secs, pairs = self.run(nb)
        return {"value": pairs / secs, "unit": "updates/s", "cores": self.workers,
                "kind": self.kind,
                "sample": f"first {nb} of {self.nb_total} batches of epoch 0 ({pairs} pair "
                          f"updates, {secs:.1f}s, {self.workers} worker threads, Philox "
                          f"negatives injected)",
                "sec_per_epoch_extrapolated": secs * self.nb_total / nb}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def config_block(cfg_name, n, nnz, world):
    """`config` of both arms (identical keys and values for the same run)."""
    gen, kw, kind, d, b, s, lr, epochs = CONFIGS[cfg_name]
    return {"workload": WORKLOAD_NAMES[cfg_name], "config_id": cfg_name, "n": n, "nnz": nnz,
            "dim": d, "batch": b, "negatives": s, "lr": lr, "force_model": kind,
            "epochs_schedule": epochs, "sampler": "philox", "init": "U(-1,1) from Rng(1, 0)",
            "arithmetic": "fp64 pair math and accumulation (the reference's operation order), "
                          "fp32 Z",
            "parallelism": f"vertex shards x{world}" if world > 1 else "1 GPU",
            "step": "one epoch (all batches) of train()"}


def bench_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import pyoracle as P

    cfg_name = args.config
    _, _, kind, d, b, s, lr, epochs = CONFIGS[cfg_name]
    rkind, graph, n, nnz = reference_graph(cfg_name)
    z0 = np.zeros((n, d), np.float32)
    P.oracle().orc_random_embedding(n, d, 1, z0)  # U(-1,1) from Rng(1, 0), A.5
    ref = ReferenceCPU(rkind, graph, n, z0, cfg_name)
    # each step: a bounded sample of the epoch (the whole run within minutes)
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    nb = ref.size_for(per_step)
    for _ in range(args.warmup):  # untimed warm-up samples (a few batches each)
        ref.run(min(nb, 4))
    runs = [ref.measure(nb) for _ in range(max(1, args.steps))]
    v = float(np.median([r["value"] for r in runs]))
    pairs = nnz + n * s
    out = {
        "impl": "reference", "metric": "edge+neg-sample updates/sec (d=128)" if d == 128 else
        "edge+neg-sample updates/sec", "value": v, "unit": "updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * pairs / v, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(cfg_name, n, nnz, 1),
        "sec_per_epoch": pairs / v,
        "cpu_baseline": {k: runs[0][k] for k in ("cores", "kind", "sample")} | {
            "value": v, "unit": "updates/s"},
        "e2e": {"value": v, "unit": "updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    return 0


def timed_epochs(f2v, dev, cfg, args, local, world):
    """K device-resident epochs in one train_epochs call after W warm-up
    epochs; CUDA events on the library stream (max over ranks)."""
    dev.train_epochs(cfg, 0, args.warmup)  # untimed warm-up epochs
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    f2v._lib.f2v_kernel_launches(dev._h, 1)
    with ClockSampler(local) as clk:
        t_wall = time.perf_counter()
        dev.train_epochs(cfg, args.warmup, args.steps)  # K timed epochs, one call
        t_wall = time.perf_counter() - t_wall
    t = dev.last_timing()
    dev_ms, kern_ms, nk = t["device_ms"], t["epoch_kernel_ms"], t["epoch_kernels"]
    assert nk == args.steps, (nk, args.steps)
    launches = f2v._lib.f2v_kernel_launches(dev._h, 0)
    if world > 1:
        import torch
        import torch.distributed as dist
        tt = torch.tensor([dev_ms, kern_ms], device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dev_ms, kern_ms = float(tt[0].item()), float(tt[1].item())
    return dev_ms, kern_ms, nk, launches, clk.summary(), t_wall


def roofline(cfg_name, precision, n, nnz, d, b, s, kern_ms_per_launch, world):
    algo = algorithmic_bytes(n, nnz, d, min(b, n), s)
    peak, peak_kind = hbm_peak()
    achieved = algo / (kern_ms_per_launch / 1e3) / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": peak * world, "unit": "GB/s",
            "frac": achieved / (peak * world),
            "traffic": ncu_traffic(f"{cfg_name}_{precision}") if world == 1 else None,
            "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" + (
                f" x {world} GPUs" if world > 1 else "") if peak_kind == "measured"
            else "fallback 6650 GB/s (B200_PROFILING.md)",
            "algorithmic_bytes_per_launch": algo,
            "kernel_ms_per_launch": kern_ms_per_launch}


PRECISION_DTYPE = {"exact": "f64",  # fp64 pair math + accumulation, as the reference
                   "fast": "f32 pair math / f64 accumulate"}


def bench_b200(args):
    import paper_2009_10035_b200 as f2v

    rank, world, local = dist_env()
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    cfg_name = args.config
    _, _, kind, d, b, s, lr, epochs = CONFIGS[cfg_name]
    g = make_graph(f2v, cfg_name)
    n, nnz = g.num_vertices(), g.num_edges()
    # epochs schedule long enough that warm-up and timed epochs each get their
    # own epoch index (own Fisher-Yates perm and negatives); lr is constant.
    cfg = f2v.TrainConfig(dim=d, batch=b, negatives=s, lr=lr,
                          epochs=args.warmup + args.steps,
                          model=f2v.ForceModel(f2v.ForceKind.parse(kind)), seed=1,
                          monitor_loss=False, sampler="philox", precision=args.precision)
    # F2V_BENCH_SHARDED=1 runs the sharded code path at world 1 as well
    sharded = world > 1 or bool(os.environ.get("F2V_BENCH_SHARDED"))
    if sharded:
        # vertex-partitioned shards: each GPU runs its
        # rows and stores every updated row into all replicas over NVLink
        from paper_2009_10035_b200.dist import ShardedDevice
        sd = ShardedDevice(rank, world, local)
        sd.setup(g, dim=d, seed=1)  # the configs' U(-1,1) from Rng(seed, 0)
        dev = sd.dev
        cfg = dataclasses.replace(cfg, shards=world)
    else:
        sd = None
        dev = f2v.Device(local)
        dev.upload_graph(g)
        dev.uniform_embedding(n, d, 1, -1.0, 1.0)  # the configs' U(-1,1) from Rng(seed, 0)
    z_start = dev.get_embedding() if args.precision == "exact" and not args.no_fast else None
    dev_ms, kern_ms, nk, launches, clocks, t_wall = timed_epochs(f2v, dev, cfg, args, local,
                                                                 world)
    z = dev.get_embedding()
    assert np.all(np.isfinite(z)), "non-finite embedding"
    pairs = nnz + n * s
    # the G shards split ONE epoch of the whole graph: total work is fixed
    value = pairs * args.steps / (dev_ms / 1e3)
    ms_per_step = dev_ms / args.steps
    roof = roofline(cfg_name, args.precision, n, nnz, d, b, s, kern_ms / nk, world)
    if world > 1:  # the fused row exchange: every GPU stores its rows into G-1 replicas
        xbytes = (world - 1) * (n // world) * 4 * d
        roof["nvlink"] = {"bytes_per_gpu_per_epoch": xbytes,
                          "achieved_GBps": xbytes / (kern_ms / nk / 1e3) / 1e9,
                          "peak_GBps": 900.0, "peak_source": "NVLink 5 nominal per direction"}
    fast = None
    if z_start is not None:  # the same epochs with fp32 pair math (precision="fast")
        dev.set_embedding(z_start) if not sharded else None
        cfg_f = dataclasses.replace(cfg, precision="fast")
        f_ms, f_kms, f_nk, _, f_clk, _ = timed_epochs(f2v, dev, cfg_f, args, local, world)
        fast = {"value": pairs * args.steps / (f_ms / 1e3), "unit": "updates/s",
                "ms_per_step": f_ms / args.steps, "dtype": PRECISION_DTYPE["fast"],
                "roofline": roofline(cfg_name, "fast", n, nnz, d, b, s, f_kms / f_nk, world),
                "clocks": f_clk,
                "note": "precision='fast': fp32 dot/distance and force term, fp32 8-pair "
                        "block sums, fp64 per-vertex accumulation; not the headline"}
    # ------------------------------------- per-step all-gather baseline
    # the same epochs run step by step (grad -> ncclAllGather of the updated
    # rows -> scatter), the reference's synchronisation granularity: what the
    # fused dataflow kernel is measured against (SURVEY.md 8(e) ladder step 1)
    per_step = None
    if not args.no_per_step:
        try:
            from paper_2009_10035_b200.dist import AllgatherDevice
            ag = AllgatherDevice(rank, world, local)
            ag.setup(g, dim=d, seed=1)
            cfg_ag = dataclasses.replace(cfg, shards=world)
            ag.train_epochs(cfg_ag, 0, 1)  # warm-up epoch
            ks = max(1, min(args.steps, 2))
            ag.train_epochs(cfg_ag, 1, ks)
            t_ag = ag.last_timing()["device_ms"]
            if world > 1:
                import torch
                import torch.distributed as dist
                tt = torch.tensor([t_ag], device=f"cuda:{local}")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t_ag = float(tt.item())
            ag.close()
            per_step = {"value": pairs * ks / (t_ag / 1e3), "unit": "updates/s",
                        "ms_per_step": t_ag / ks, "epochs": ks,
                        "exchange": f"ncclAllGather of every step's updated rows, world {world}",
                        "dtype": PRECISION_DTYPE[args.precision],
                        "note": "f2v_train_epochs_allgather: per step one grad kernel "
                                "(one warp per batch row), the all-gather, a vote and a "
                                "scatter kernel; same results as the fused epoch kernel"}
        except Exception as ex:  # reported, not hidden
            per_step = {"value": None, "error": str(ex)}
    # ------------------------------------------------------------ e2e
    import torch
    h_row = torch.from_numpy(g.row_offsets).pin_memory().numpy()
    h_col = torch.from_numpy(g.col_indices).pin_memory().numpy()
    h_z0 = torch.empty((n, d), dtype=torch.float32).pin_memory().numpy()
    h_z = torch.empty((n, d), dtype=torch.float32).pin_memory().numpy()
    dev.uniform_embedding(n, d, 1, -1.0, 1.0)
    h_z0[:] = dev.get_embedding()
    e2e_steps = max(1, min(args.steps, 3))
    g_pinned = f2v.CsrGraph(h_row, h_col)

    cfg_e2e = f2v.TrainConfig(dim=d, batch=b, negatives=s, lr=lr, epochs=epochs,
                              model=cfg.model, seed=1, monitor_loss=False, sampler="philox",
                              precision=args.precision)

    if sharded:
        cfg_e2e = dataclasses.replace(cfg_e2e, shards=world)

    def e2e_once():
        if sharded:  # the public sharded API, from host buffers
            s2 = ShardedDevice(rank, world, local)
            s2.setup(g_pinned, h_z0)
            s2.train_epochs(cfg_e2e)
            out = np.ascontiguousarray(h_z)
            f2v._lib.f2v_get_embedding(s2.dev._h, out)
            s2.close()
            return out
        dev.upload_graph(g_pinned)
        dev.set_embedding(h_z0)
        dev.train_epochs(cfg_e2e, 0, 0)
        out = np.ascontiguousarray(h_z)
        f2v._lib.f2v_get_embedding(dev._h, out)
        return out
    e2e_once()  # warm
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_once()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        tt = torch.tensor([e2e_s], device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    e2e_val = pairs * epochs / e2e_s
    h2d = h_row.nbytes + h_col.nbytes + h_z0.nbytes
    d2h = h_z.nbytes
    dev.close()
    if rank != 0:
        return 0
    conf = config_block(cfg_name, n, nnz, world)
    if args.precision != "exact":
        conf["arithmetic"] = PRECISION_DTYPE[args.precision]
    conf["l2"] = "inputs larger than L2 (Z 2x%d MB + CSR %d MB > 126 MB)" % (
        n * d * 4 >> 20, (nnz * 4 + n * 8) >> 20)
    out = {
        "metric": "edge+neg-sample updates/sec (d=128)" if d == 128 else
        "edge+neg-sample updates/sec", "value": value, "unit": "updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": PRECISION_DTYPE[args.precision], "data": "synthetic",
        "config": conf,
        "sec_per_epoch": ms_per_step / 1e3,
        "roofline": roof,
        "e2e": {"value": e2e_val, "unit": "updates/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "step": f"one train() of the {epochs}-epoch schedule via the public API "
                        f"(CSR + Z copied in from pinned host buffers the bench allocates, "
                        f"Z copied out): {e2e_s * 1e3:.1f} ms"},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "wall_s_timed_region": t_wall,
    }
    if fast is not None:
        out["fast"] = fast
    if per_step is not None:
        out["per_step_baseline"] = per_step
    if world == 1 and not args.no_cpu_baseline:
        try:
            import pyoracle as P
            if P.reference_available():
                graph, rk = P.RefGraph.from_csr(g.row_offsets, g.col_indices), "reference"
            else:
                graph, rk = (g.row_offsets, g.col_indices), "port"
            ref = ReferenceCPU(rk, graph, n, h_z0, cfg_name)
            out["cpu_baseline"] = ref.measure(ref.size_for(args.cpu_budget))
        except Exception as ex:  # reported, not hidden
            out["cpu_baseline"] = {"value": None, "error": str(ex)}
    print(json.dumps(out), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--precision", default="exact", choices=["exact", "fast"])
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fast", action="store_true", help="skip the precision='fast' run")
    ap.add_argument("--no-per-step", action="store_true",
                    help="skip the per-step ncclAllGather baseline")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        log("note: warm-up raised to the contract minimum of 3")
        args.warmup = 3
    if args.impl == "reference":
        return bench_reference(args)
    return bench_b200(args)


if __name__ == "__main__":
    sys.exit(main())
