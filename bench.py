#!/usr/bin/env python
"""Benchmark of the sparse hot path (BASELINE.json metric) -- one JSON line.

Default workload (BASELINE configs[4], "cfg5", the largest config; the one
that carries the metric's "GNN epoch time"): a 2-layer GraphSAGE-mean
training epoch -- train()'s loop body, gnn.hpp:427-435 -- on an R-MAT graph
with 2^22 nodes, N*25 samples symmetrised + self loops, dedup (201.75M nnz),
X 2^22 x 128 N(0,1), hidden 128, 16 classes, uniform labels, every node in
the mask.  One *step* = one epoch: 2 forward SpMMs (mean), 1 backward SpMM
through the cached mean operand, the dense products and glue, SGD.  At N=1
the whole graph is on one GPU; at N>1 its rows are partitioned over the
ranks (nnz + 30*rows cost) with NCCL all-gathers of the feature blocks and an
all-reduce of the weight gradients (csrc/dist.cu through sgnn_dist_*).

  value      = 3 * 2*nnz*K / epoch time  [GFLOP/s over the epoch's 3 SpMMs],
               median over the K timed epochs of the per-epoch device time
               (CUDA events, max over ranks); inputs resident in HBM; the
               inputs are larger than L2 (no flush needed)
  epoch_ms   = that epoch time (the metric's "GNN epoch time")
  e2e        = the same epochs through the public API with the rank's feature
               rows uploaded from pinned host memory every epoch and the
               epoch's (loss, accuracy) read back
  roofline   = algorithmic bytes of the 3 SpMM calls / their event-timed
               duration vs the measured HBM bandwidth (MEASURED_PEAKS.json);
               dram_frac / l2_frac from the ncu capture (profiles/traffic.json)

--impl reference: the reference's own CPU implementation of the epoch
(oracle/_ref, compiled from /root/reference/proj): each step is a row sample
of the SAGE epoch made of the reference's own calls (ref_shim.cpp
ref_sage_sample_*), sized so the run ends within minutes.
--gpus N without torchrun: the script re-executes itself as N ranks.
--workload cfg1|cfg2|cfg3|cfg4: the other BASELINE configs.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpMM/FusedMM GFLOP/s (2·nnz·K) and % of HBM roofline; GNN epoch time"
FALLBACK_HBM = 6650.0
LR = 0.05

# Pure-gather ceiling on cfg2's own column sequence (512-byte rows, 128 MB
# table): scripts/probes/gather_probe.cu on the B200, 16 CTAs/SM x U=4 best.
GATHER_PROBE_CFG2_GBPS = 20201.0


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--plan", type=str, default="", help="JSON plan params override (cfg2)")
    p.add_argument("--workload", choices=("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"), default="cfg5",
                   help="cfg5 (default, the headline: GraphSAGE-mean epoch, 1 GPU or row-partitioned) | "
                        "cfg1 small ER SpMM | cfg2 SpMM fwd+bwd | cfg3 GCN layer | cfg4 FusedMM/SDDMM")
    p.add_argument("--row-weight", type=int, default=30, help="cfg5 partition cost nnz + w*rows")
    p.add_argument("--ref-budget", type=float, default=150.0, help="seconds of CPU work for --impl reference")
    p.add_argument("--loopback", type=int, default=0,
                   help="cfg5: run P virtual ranks on one GPU (per-rank balance, not a throughput number)")
    p.add_argument("--dry-run-dist", action="store_true", help=argparse.SUPPRESS)
    return p.parse_args(argv)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md 6.65 TB/s)"


def spmm_bytes(m, nnz, k):
    """Algorithmic bytes: CSR arrays + feature gathers + output."""
    return 8 * (m + 1) + 8 * nnz + 4 * nnz * k + 4 * m * k


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        pass
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def load_traffic(workload):
    """ncu per-launch figures of the dominant kernel (profiles/traffic.json):
    dram bytes, the kernel's ncu duration, lts__throughput %, L2 hit %."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


def traffic_fields(workload, t_kernel_ms, peak):
    """roofline.traffic, dram_frac, l2_frac for one launch of `workload`'s
    dominant kernel timed at t_kernel_ms here (ncu's own duration is cold-cache
    and serialised, so the DRAM rate uses this run's duration)."""
    d = load_traffic(workload)
    if not d:
        return {"traffic": None, "dram_frac": None, "l2_frac": None}
    tb = int(d["dram_bytes_per_launch"])
    out = {"traffic": tb,
           "dram_frac": round(tb / (t_kernel_ms * 1e-3) / 1e9 / peak, 4) if t_kernel_ms else None,
           "l2_frac": round(float(d["lts_throughput_pct"]) / 100, 4) if d.get("lts_throughput_pct") is not None else None,
           "l2_hit_pct": d.get("l2_hit_pct"), "ncu_source": d.get("source")}
    return out


# ------------------------------------------------------------- rank spawning
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int, argv, check_gpus: bool = True) -> int:
    """--gpus N outside torchrun: re-execute this script as N ranks (one
    process per GPU, RANK/LOCAL_RANK/WORLD_SIZE/MASTER_* in the environment,
    rendezvous on 127.0.0.1).  Fails loudly when fewer than N GPUs are
    visible.  Returns the worst exit code."""
    if check_gpus:
        import torch
        have = torch.cuda.device_count()
        if have < n:
            print(json.dumps({"error": f"--gpus {n} requested but only {have} CUDA device(s) are visible"}),
                  flush=True)
            return 2
    port = str(_free_port())
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + list(argv), env=env))
    return max(p.wait() for p in procs)


def dry_run_dist(args):
    """The spawn path without GPUs (tests): every rank joins a gloo group,
    the max over ranks is taken like a timed run, rank 0 prints the line."""
    import torch
    import torch.distributed as dist
    ws, rank, _ = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": ws, "max_over_ranks": float(t[0]), "workload": args.workload}),
              flush=True)


# ------------------------------------------------------------------- cfg5 (headline)
def cfg5_inputs(seed):
    from paper_2403_14853_b200 import graphs
    w = graphs.cfg5(seed)
    n, k = w.n_rows, w.k
    x = graphs.normal(n * k, 0.0, 1.0, seed, stream=51).reshape(n, k)
    labels = (np.arange(n, dtype=np.uint64) * 2654435761 % 16).astype(np.uint32)  # uniform over 16 classes
    mask = np.ones(n, np.uint8)  # every node (io.hpp:367)
    return w, x, labels, mask


def cfg5_weights(seed, k=128, hidden=128, classes=16):
    """Glorot-uniform w1, w2, w1_self, w2_self (gnn.hpp:75-99 shapes), host fp32."""
    from paper_2403_14853_b200 import graphs

    def glorot(r, c, stream):
        lim = float(np.sqrt(6.0 / (r + c)))
        return graphs.uniform(r * c, -lim, lim, seed, stream=stream).reshape(r, c)
    return glorot(k, hidden, 61), glorot(hidden, classes, 62), glorot(k, hidden, 63), glorot(hidden, classes, 64)


def cfg5_config(w, ws, bounds, extra=None):
    c = {"workload": "cfg5: 2-layer GraphSAGE-mean training epoch (train() loop body, gnn.hpp:427-435), R-MAT 2^22 "
                     "N*25 samples symmetrised + self loops (dedup), X N(0,1) 2^22x128, hidden 128, 16 classes, "
                     "uniform labels, mask = all nodes",
         "n_rows": w.n_rows, "nnz": w.nnz, "K": w.k, "hidden": 128, "classes": 16, "seed": w.seed,
         "rmat": "(0.57,0.19,0.19,0.05), no permutation", "lr": LR,
         "l2": "inputs larger than L2 (X 2 GiB, CSR 1.6 GB, activations 2 GiB each): no flush between steps",
         "parallelism": ("1 GPU (whole graph)" if ws == 1 else
                         f"1D row partition x{ws} (nnz + 30*rows cost), NCCL all-gather-v of feature blocks "
                         "(grouped send/recv, no padding) + all-reduce of weight gradients"),
         "partition_bounds": [int(b) for b in bounds]}
    if extra:
        c.update(extra)
    return c


def run_cfg5(args):
    import torch

    from paper_2403_14853_b200 import dist as sdist
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    tdist = None
    comm = None
    if ws > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=dev)
        comm = sdist.Comm.from_torch()
    t0 = time.time()
    w, x_np, labels, mask = cfg5_inputs(args.seed)
    gen_s = time.time() - t0
    W, K = max(3, args.warmup), max(1, args.steps)
    e2e_steps = 0 if args.no_e2e else min(K, 20)
    t0 = time.time()
    eng = sdist.DistSage.from_graph(comm, w.row_ptr, w.col_idx, w.values, x_np, labels, mask, 128, 16,
                                    "sage-mean", row_weight=args.row_weight, max_epochs=W + K)
    w1, w2, w1s, w2s = cfg5_weights(args.seed)
    eng.set_weights(w1, w2, w1s, w2s)
    setup_s = time.time() - t0
    stream = torch.cuda.current_stream()
    eng.epochs(W, LR)
    torch.cuda.synchronize()
    if tdist:
        tdist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(_nvml_index(local)) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        eng.epochs(K, LR)
        e1.record(stream)
        torch.cuda.synchronize()
    if tdist:
        tdist.barrier()
    loss, acc, times = eng.stats(W, K)
    total_ms = e0.elapsed_time(e1)
    # per-epoch max over ranks, then the median; the bracketed total too
    per = torch.tensor(np.concatenate([times[:, 0], times[:, 1], times[:, 2], times[:, 3], [total_ms]]),
                       dtype=torch.float64, device=dev)
    if tdist:
        tdist.all_reduce(per, op=tdist.ReduceOp.MAX)
    per = per.cpu().numpy()
    ep_max, sp_max, comp_max, ex_max, total_max = per[:K], per[K:2 * K], per[2 * K:3 * K], per[3 * K:4 * K], per[-1]
    epoch_ms = float(np.median(ep_max))
    nnz, k = w.nnz, w.k
    flops = 3 * 2 * nnz * k
    value = flops / (epoch_ms * 1e-3) / 1e9
    peak, peak_src = peaks()
    # roofline of this rank's SpMM calls (worker + fixups + mean epilogue)
    sp_ms = float(np.median(times[:, 1]))
    rows, bnnz = eng.rows, eng.nnz
    alg = 3 * spmm_bytes(rows, bnnz, k)
    achieved = alg / (sp_ms * 1e-3) / 1e9
    per_call = [float(np.median(times[:, j])) for j in (4, 5, 6)]
    tf = traffic_fields("cfg5", per_call[0], peak)
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": tf["traffic"], "peak_source": peak_src,
            "dram_frac": tf["dram_frac"], "l2_frac": tf["l2_frac"], "l2_hit_pct": tf.get("l2_hit_pct"),
            "alg_bytes_per_launch": alg // 3, "spmm_ms_per_call": [round(t, 4) for t in per_call],
            "note": "per SpMM call of rank 0 (worker + fixups + mean epilogue; events on the engine's stream): "
                    "achieved = algorithmic bytes (CSR + gathered X rows + output, SURVEY 8d) / duration; "
                    "traffic / dram_frac / l2_frac = ncu dram bytes, DRAM rate at this run's duration, "
                    "lts__throughput of the layer-1 SpMM worker (profiles/traffic.json)"}
    out = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": ws, "steps": K, "warmup": W,
        "ms_per_step": round(epoch_ms, 4), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (seeded R-MAT, BASELINE cfg5 shapes; paper datasets not available offline)",
        "config": cfg5_config(w, ws, eng.bounds),
        "epoch_ms": round(epoch_ms, 4), "epoch_ms_mean": round(total_max / K, 4),
        "spmm_ms": round(float(np.median(sp_max)), 4), "compute_ms": round(float(np.median(comp_max)), 4),
        "exchange_ms": round(float(np.median(ex_max)), 4),
        "dense_ms": round(float(np.median(times[:, 7])), 4),
        "sparse_gflops": round(flops / (float(np.median(sp_max)) * 1e-3) / 1e9, 2),
        "loss_first_last": [round(float(loss[0]), 6), round(float(loss[-1]), 6)],
        "accuracy_last": round(float(acc[-1]), 6),
        "roofline": roof,
        "gpu_launches": K * (CFG5_LAUNCHES_PER_EPOCH + (2 if ws > 1 else 0)),
        "gen_s": round(gen_s, 2), "setup_s": round(setup_s, 2),
    }
    out["clocks"] = clk.summary()
    if e2e_steps:
        out["e2e"] = cfg5_e2e(eng, x_np, e2e_steps, flops, dev, tdist)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            cb = cfg5_reference_run(w, x_np, labels, mask, steps=3, warmup=1, budget_s=25.0)
            cb = {kk: cb[kk] for kk in ("value", "unit", "cores", "kind", "sample", "cpu_model", "ms_per_step",
                                         "flavour")}
        except Exception as ex:  # noqa: BLE001
            cb = {"error": repr(ex)}
        out["cpu_baseline"] = cb
    eng.close()
    if comm:
        comm.close()
    if tdist:
        tdist.barrier()
        tdist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


# our kernels launched per cfg5 epoch at N=1 (ncu launch list, profiles/r02o_cfg5_launches.json):
# 3 SpMMs (worker + 2 fixups each; the mean divide is in the epilogue), 2 tensor-core
# products (relu in the first one's epilogue), head, rank stats, wgrad + finish,
# relu-backward, sgd, epoch record; at N > 1 also the two remote-row ds2 passes
CFG5_LAUNCHES_PER_EPOCH = 18


def _nvml_index(local):
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    if cvd:
        ids = cvd.split(",")
        if local < len(ids) and ids[local].strip().isdigit():
            return int(ids[local])
    return local


def cfg5_e2e(eng, x_np, steps, flops, dev, tdist):
    """Public-API epochs with host buffers: every epoch uploads the rank's
    feature rows from pinned host memory (copy stream, double-buffered: the
    upload of epoch i+1 overlaps epoch i) and reads the epoch's (loss,
    accuracy) back into pinned host memory."""
    import torch
    r0, rows = eng.r0, eng.rows
    hx = torch.from_numpy(np.ascontiguousarray(x_np[r0:r0 + rows])).pin_memory()
    hres = torch.zeros(2 * steps, dtype=torch.float64).pin_memory()
    nb = 2
    xb = [torch.empty_like(hx, device=dev) for _ in range(nb)]
    comp = torch.cuda.current_stream()
    up = torch.cuda.Stream()
    free = [torch.cuda.Event() for _ in range(nb)]
    for e in free:
        e.record(comp)
    eng.reset()

    def upload(i):
        b = i % nb
        with torch.cuda.stream(up):
            up.wait_event(free[b])
            xb[b].copy_(hx, non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(up)
        return ready

    torch.cuda.synchronize()
    if tdist:
        tdist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    up.wait_stream(comp)
    ready = upload(0)
    for i in range(steps):
        comp.wait_event(ready)
        eng.set_features(xb[i % nb])  # device copy into [a1 | X_r] (P>1: also the gathered buffer, re-exchanged)
        eng.epochs(1, LR)
        free[i % nb].record(comp)
        if i + 1 < steps:
            ready = upload(i + 1)
        eng.stats_copy(i, 1, hres.data_ptr() + 16 * i)
    comp.wait_stream(up)
    e1.record(comp)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if tdist:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": round(flops * steps / (ms * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
            "h2d_bytes_per_step": int(hx.numel() * 4), "d2h_bytes_per_step": 16,
            "ms_per_step": round(ms / steps, 4), "steps": steps, "loss_last": float(hres[2 * steps - 2]),
            "note": "graph + weights resident (like the reference's TrainingCache / model); each epoch uploads this "
                    "rank's feature rows from pinned host memory on a copy stream (double-buffered, overlapping the "
                    "previous epoch) and copies the epoch's (loss, accuracy) to pinned host memory"}


def cfg5_reference_run(w, x_np, labels, mask, steps, warmup, budget_s, flavours=None):
    """The reference's CPU epoch (oracle/_ref) on all host threads.  A full
    cfg5 epoch takes ~1 min on 8 cores (build_cache ~50 s once), so each
    step is a ROW SAMPLE of the SAGE epoch made of the reference's own calls
    (ref_shim.cpp ref_sage_sample_*), all columns (rows R: a seeded uniform sample of n/f rows, whose nnz share
    is within a few % of 1/f); f is set from a calibration run so that warmup + steps fit
    the budget.  value = 3 * 2 * nnz(R) * K / sample time."""
    from oracle import ref
    flav = flavours or ref.flavours()
    if not flav:
        return None
    n, k = w.n_rows, w.k
    rp = np.asarray(w.row_ptr, np.uint64)
    deg = np.diff(rp.astype(np.int64)).astype(np.float32)
    mvals = (np.asarray(w.values, np.float32) / deg[np.asarray(w.col_idx, np.int64)]).astype(np.float32)
    winit = np.concatenate([a.ravel() for a in cfg5_weights(w.seed)]).astype(np.float32)

    def sample(f):
        # uniform random rows (seeded): R-MAT ids are not permuted, so strided
        # rows would over-sample the hubs (ids with many zero low bits)
        rows = np.sort(np.random.default_rng(12345).choice(n, max(1, n // f), replace=False))
        d = np.diff(rp.astype(np.int64))[rows]
        srp = np.zeros(len(rows) + 1, np.uint64)
        srp[1:] = np.cumsum(d)
        starts = rp[rows].astype(np.int64)
        idx = (np.repeat(starts - np.concatenate([[0], np.cumsum(d)[:-1]]), d) + np.arange(int(srp[-1]))).astype(np.int64)
        return rows, srp, idx

    def make(f, fl):
        rows, srp, idx = sample(f)
        ci = np.asarray(w.col_idx)[idx]
        s = ref.SageSample("sage-mean", n, (srp, ci, np.asarray(w.values, np.float32)[idx]), (srp, ci, mvals[idx]),
                           x_np, x_np[rows], x_np, labels[rows], mask[rows], 128, 16, winit, LR, 0, fl)
        return s, len(rows), int(srp[-1])

    # calibrate flags and size on a small sample
    f0 = 64
    best, best_t = None, None
    for fl in flav:
        s, _, _ = make(f0, fl)
        s.epoch()  # first touch
        t0 = time.perf_counter()
        s.epoch()
        t = time.perf_counter() - t0
        s.close()
        if best_t is None or t < best_t:
            best, best_t = fl, t
    per_step = budget_s / (steps + warmup)
    f = max(1, int(np.ceil(best_t * f0 / per_step)))
    s, n_r, nnz_r = make(f, best)
    for _ in range(warmup):
        s.epoch()
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        s.epoch()
        ts.append(time.perf_counter() - t0)
    s.close()
    med = float(np.median(ts))
    from oracle.ref import FLAVOURS
    return {"value": round(3 * 2 * nnz_r * k / med / 1e9, 4), "unit": "GFLOP/s", "cores": os.cpu_count() or 1,
            "kind": "reference", "cpu_model": cpu_model(), "ms_per_step": round(med * 1e3, 3), "steps": steps,
            "flavour": f"g++ {FLAVOURS[best][1]}",
            "sample": (f"row sample of the cfg5 SAGE-mean epoch: {n_r} of {n} rows (seeded uniform), "
                       f"{nnz_r} of {w.nnz} nnz, the epoch's reference calls (spmm x3, matmul/matmul_tn/matmul_nt, "
                       f"relu, softmax_xent, masked_accuracy, relu_backward, sgd_step) on those rows; median of "
                       f"{steps} after {warmup} warm-up"),
            "full_epoch_ms_est": round(med * 1e3 * n / n_r, 1)}


def run_reference_cfg5(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    w, x_np, labels, mask = cfg5_inputs(args.seed)
    cb = cfg5_reference_run(w, x_np, labels, mask, steps=max(1, args.steps), warmup=max(0, args.warmup),
                            budget_s=args.ref_budget)
    if cb is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference at build time)"}))
        return
    out = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "GFLOP/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["ms_per_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded R-MAT, BASELINE cfg5 shapes)",
        "config": cfg5_config(w, 1, [0, w.n_rows], {"l2": "n/a (CPU)", "parallelism": "host threads"}),
        "epoch_ms_est": cb["full_epoch_ms_est"],
        "cpu_baseline": {"value": cb["value"], "unit": "GFLOP/s", "cores": cb["cores"], "kind": "reference",
                         "sample": cb["sample"], "cpu_model": cb["cpu_model"], "flavour": cb["flavour"]},
        "e2e": {"value": cb["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def run_loopback_cfg5(args):
    """P virtual ranks of the cfg5 partition on one GPU (serial, one stream):
    each rank's compute time per epoch -- the partition's balance -- and the
    exchange bytes each rank would receive."""
    import torch

    from paper_2403_14853_b200 import dist as sdist
    P = args.loopback
    torch.cuda.set_device(0)
    w, x_np, labels, mask = cfg5_inputs(args.seed)
    comm = sdist.Comm.loopback(P)
    bounds = sdist.row_partition(w.row_ptr, P, args.row_weight)
    engs = [sdist.DistSage.from_graph(comm, w.row_ptr, w.col_idx, w.values, x_np, labels, mask, 128, 16,
                                      "sage-mean", rank=r, bounds=bounds, symmetric=True, max_epochs=64)
            for r in range(P)]
    ws_ = cfg5_weights(args.seed)
    for e in engs:
        e.set_weights(*ws_)
    W, K = max(1, args.warmup), max(1, args.steps)
    sdist.DistSage.epochs_group(engs, W + K, LR)
    torch.cuda.synchronize()
    comp = np.array([np.median(e.stats(W, K)[2][:, 2]) for e in engs])
    spmm = np.array([np.median(e.stats(W, K)[2][:, 1]) for e in engs])
    loss = engs[0].stats(W, K)[0]
    rows = np.diff(bounds.astype(np.int64))
    recv = [(w.n_rows - int(r)) * (128 + 16) * 4 for r in rows]  # h1 + grad all-gathers per epoch (X gathered once)
    print(json.dumps({"loopback_ranks": P, "row_weight": args.row_weight, "bounds": [int(b) for b in bounds],
                      "rank_compute_ms": [round(float(c), 3) for c in comp],
                      "rank_spmm_ms": [round(float(c), 3) for c in spmm],
                      "max_over_mean": round(float(comp.max() / comp.mean()), 4),
                      "recv_bytes_per_epoch": recv, "loss_last": float(loss[-1]),
                      "nnz_per_rank": [int(e.nnz) for e in engs]}), flush=True)
    for e in engs:
        e.close()
    comm.close()


class ClockSampler:
    """Samples SM clocks and clock-event reasons via NVML during the timed region."""
    NAMES = {0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
             0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self.stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                try:
                    bits = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    bits = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for b, n in self.NAMES.items():
                    if bits & b:
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self.stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def spmm_launches(plan, row_ptr):
    """Kernels one SpMM / FusedMM call with `plan` launches: the worker, the
    per-row fixup when rows are split, and the long-row fixup when a split
    row has more than SGNN_FIXUP_LONG (32) segments of 256 nonzeros."""
    deg = np.diff(np.asarray(row_ptr, np.uint64).astype(np.int64))
    split = plan.stats["split_rows"] > 0
    long_rows = split and bool((deg > 32 * 256).any())
    return 1 + int(split) + int(long_rows)



# ------------------------------------------------------------------- cfg2
def build_workload(seed):
    from paper_2403_14853_b200 import graphs
    w = graphs.cfg2(seed)
    x = graphs.normal(w.n_cols * w.k, 0.0, 1.0, seed, stream=21).reshape(w.n_cols, w.k)
    g = graphs.normal(w.n_rows * w.k, 0.0, 1.0, seed, stream=22).reshape(w.n_rows, w.k)
    return w, x, g


def config_of(w, extra=None):
    c = {"workload": "cfg2: SpMM fwd + bwd (cached CSC), R-MAT 2^18 avg-deg 256 sampled, dedup",
         "n_rows": w.n_rows, "nnz": w.nnz, "K": w.k, "reduce": "sum", "values": "1.0",
         "X,dC": "N(0,1)", "rmat": "(0.57,0.19,0.19,0.05), no permutation, N*256 samples",
         "seed": w.seed, "l2": "flushed between steps (256 MiB write + 256 MiB read), flush not timed"}
    if extra:
        c.update(extra)
    return c


def cpu_reference_run(w, x, g, steps, warmup, budget_s=150.0, flavours=None):
    """Times the reference's own CPU path (oracle/_ref) on all host threads.
    Picks the fastest (flags, kernel) pair like BASELINE.md section 2, then
    times `steps` fwd+bwd steps; if that would exceed the budget, each step is
    a row sample of the workload (every f-th 64-row block of A, all columns)."""
    import numpy as np

    from oracle import ref
    flav = flavours or ref.flavours()
    if not flav:
        return None
    cores = os.cpu_count() or 1
    rp, ci, v = w.row_ptr, w.col_idx, w.values

    def make(rp_, ci_, v_):
        return {f: ref.Bench(rp_, ci_, v_, w.n_cols, x, g[: len(rp_) - 1], 0, f) for f in flav}

    def sample(frac):
        # seeded uniform rows: R-MAT ids are not permuted, so strided row
        # blocks would over-sample the hubs
        m = w.n_rows
        rows = np.sort(np.random.default_rng(12345).choice(m, max(1, m // frac), replace=False))
        deg = np.diff(rp.astype(np.int64))[rows]
        srp = np.zeros(len(rows) + 1, np.uint64)
        srp[1:] = np.cumsum(deg)
        idx = np.concatenate([np.arange(rp[i], rp[i + 1], dtype=np.int64) for i in rows]) if len(rows) else np.zeros(0, np.int64)
        return srp, ci[idx], v[idx]

    frac = 1
    benches = make(rp, ci, v)
    best, best_t = None, None
    for f, b in benches.items():
        for spec in (False, True):
            dt = None
            for _ in range(3):  # the first call also pays first-touch page faults; min of 3 (noisy hosts)
                t0 = time.perf_counter()
                b.step(specialized=spec, threads=0)
                t = time.perf_counter() - t0
                dt = t if dt is None else min(dt, t)
            if best_t is None or dt < best_t:
                best, best_t = (f, spec), dt
    est = best_t * (steps + warmup)
    nnz = w.nnz
    if est > budget_s:
        frac = int(np.ceil(est / budget_s))
        srp, sci, sv = sample(frac)
        benches = {best[0]: ref.Bench(srp, sci, sv, w.n_cols, x, g[: len(srp) - 1], 0, best[0])}
        nnz = int(srp[-1])
    b = benches[best[0]]
    for _ in range(warmup):
        b.step(specialized=best[1], threads=0)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        b.step(specialized=best[1], threads=0)
        times.append(time.perf_counter() - t0)
    for bb in benches.values():
        bb.close()
    med = float(np.median(times))
    flops = 2 * (2 * nnz * w.k)
    from oracle.ref import FLAVOURS
    return {
        "value": flops / med / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": "reference",
        "cpu_model": cpu_model(), "ms_per_step": med * 1e3,
        "sample": (f"full cfg2 fwd+bwd step ({nnz} nnz)" if frac == 1 else
                   f"1/{frac} row sample of cfg2 (seeded uniform rows; {nnz} nnz) per step") +
                  f"; median of {steps} after {warmup} warm-up",
        "kernel": f"{'specialized' if best[1] else 'trusted'} spmm_into, g++ {FLAVOURS[best[0]][1]}",
        "steps": steps,
    }


def run_cfg2(args):
    import numpy as np
    import torch

    from paper_2403_14853_b200 import ops

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    t0 = time.time()
    w, x_np, g_np = build_workload(args.seed)
    gen_s = time.time() - t0
    a = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols, device=dev)
    x = torch.from_numpy(x_np).to(dev)
    g = torch.from_numpy(g_np).to(dev)
    c = torch.empty(w.n_rows, w.k, device=dev)
    dx = torch.empty(w.n_cols, w.k, device=dev)
    flush = L2Flush(dev)
    stream = torch.cuda.current_stream()

    params = json.loads(args.plan) if args.plan else {}
    torch.cuda.synchronize()
    e_t0, e_t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_t0.record()
    cache = ops.TrainingCache(a, True)          # symmetric probe + degrees
    at = cache.sum_operand()                     # device CSC, built once (counted)
    e_t1.record()
    torch.cuda.synchronize()
    cache_ms = e_t0.elapsed_time(e_t1)
    plan_f = ops.Plan(a, w.k, **params)
    plan_b = ops.Plan(at, w.k, **params)

    def step():
        ops.spmm_plan(a, x, "sum", plan_f, c)
        ops.spmm_plan(at, g, "sum", plan_b, dx)

    for _ in range(max(3, args.warmup)):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    nvml_index = local
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    if cvd:
        ids = cvd.split(",")
        if local < len(ids) and ids[local].strip().isdigit():
            nvml_index = int(ids[local])
    with ClockSampler(nvml_index) as clk:
        torch.cuda.synchronize()
        for s in range(args.steps):
            flush.zero_()
            ev[s][0].record(stream)
            ops.spmm_plan(a, x, "sum", plan_f, c)
            ev[s][1].record(stream)
            ops.spmm_plan(at, g, "sum", plan_b, dx)
            ev[s][2].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    fwd = [e[0].elapsed_time(e[1]) for e in ev]
    bwd = [e[1].elapsed_time(e[2]) for e in ev]
    per_step = [f + b for f, b in zip(fwd, bwd)]
    ms_step = float(np.median(per_step))
    if dist:
        tt = torch.tensor([ms_step], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_step = float(tt.item())
    flops_step = 2 * (2 * w.nnz * w.k)
    value = flops_step * ws / (ms_step * 1e-3) / 1e9

    # warm-L2 reference number (not the headline)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(10):
        step()
    s1.record()
    torch.cuda.synchronize()
    warm_ms = s0.elapsed_time(s1) / 10

    # BASELINE cfg2 is "sum/mean": the same step with ReduceOp::Mean (forward
    # divides by deg; the backward runs on the cached mean operand, Aᵀ with
    # 1/deg values, gnn.hpp:149-159), reported beside the sum headline
    atm = cache.mean_operand()
    plan_bm = ops.Plan(atm, w.k, **params)
    tm_f = _events_time(lambda: ops.spmm_plan(a, x, "mean", plan_f, c), 10, 3, flush)
    tm_b = _events_time(lambda: ops.spmm_plan(atm, g, "sum", plan_bm, dx), 10, 3, flush)
    mean_ms = (sum(tm_f) + sum(tm_b)) / len(tm_f)
    mean_leg = {"fwd_ms": round(sum(tm_f) / len(tm_f), 4), "bwd_ms": round(sum(tm_b) / len(tm_b), 4),
                "GFLOP/s": round(flops_step / mean_ms / 1e6, 2),
                "note": "ReduceOp::Mean step: fwd spmm(A, X, mean) (sum kernels + divide pass), bwd through "
                        "TrainingCache::mean_operand; L2 flushed between calls"}

    # roofline of the SpMM launches (worker + fixup per call)
    bytes_f = spmm_bytes(w.n_rows, w.nnz, w.k)
    bytes_b = spmm_bytes(w.n_cols, w.nnz, w.k)
    peak, peak_src = peaks()
    achieved = (bytes_f + bytes_b) * args.steps / (sum(fwd) + sum(bwd)) / 1e6  # GB/s
    pf, pb = plan_f.stats, plan_b.stats
    launches_step = spmm_launches(plan_f, w.row_ptr) + spmm_launches(plan_b, at.to_numpy()[0])
    tf = traffic_fields("cfg2", (sum(fwd) + sum(bwd)) / (2 * args.steps), peaks()[0])
    traffic = tf["traffic"]

    # parity spot check of this run's outputs (cheap; full parity lives in tests/)
    out = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": ws,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms_step, 4), "ms_per_step_mean": round((sum(fwd) + sum(bwd)) / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded R-MAT, BASELINE cfg2 shapes; paper datasets not available offline)",
        "config": config_of(w, {"parallelism": f"replicas x{ws}" if ws > 1 else "1 GPU",
                                "plan_fwd": plan_f.params, "plan_bwd": plan_b.params}),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "dram_frac": tf["dram_frac"], "l2_frac": tf["l2_frac"], "l2_hit_pct": tf.get("l2_hit_pct"),
                     "peak_source": peak_src,
                     "alg_bytes_per_launch": (bytes_f + bytes_b) // 2,
                     "traffic_GBps_at_measured_time": (round(traffic / ((sum(fwd) + sum(bwd)) / (2 * args.steps)) / 1e6, 1)
                                                       if traffic else None),
                     "gather": {
                         "bytes_per_call": w.nnz * w.k * 4,
                         "achieved_GBps": round(w.nnz * w.k * 4 * 2 * args.steps / (sum(fwd) + sum(bwd)) / 1e6, 1),
                         "probe_ceiling_GBps": GATHER_PROBE_CFG2_GBPS,
                         "frac_of_probe": round(w.nnz * w.k * 4 * 2 * args.steps / (sum(fwd) + sum(bwd)) / 1e6
                                                / GATHER_PROBE_CFG2_GBPS, 4),
                         "note": "the binding stream: X-row gathers (L2 hit 91%). probe_ceiling = pure gather "
                                 "of the same column sequence, no values/row ends, best of 6 occupancies x 3 "
                                 "depths (scripts/probes/gather_probe.cu, DESIGN 3.1)"},
                     "note": "per SpMM call (worker + fixup): achieved = algorithmic bytes (CSR + gathered X rows "
                             "+ output) / event-timed duration; gathers of hub rows hit L2 (ncu: ~91% L2 hit), so "
                             "frac > 1 and traffic (ncu dram bytes per call, profiles/traffic.json) << algorithmic"},
        "gpu_launches": launches_step * args.steps,
        "fwd_ms": round(sum(fwd) / args.steps, 4), "bwd_ms": round(sum(bwd) / args.steps, 4),
        "warm_l2_ms_per_step": round(warm_ms, 4), "transpose_ms": round(cache_ms, 3),
        "cache_build_ms": cache_build_times(a, dev), "mean": mean_leg,
        "gen_s": round(gen_s, 2),
    }
    out["clocks"] = clk.summary()

    if not args.no_e2e:
        out["e2e"] = e2e_run(a, at, w, x_np, g_np, dev, plan_f, plan_b, args, ws, dist)

    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_reference_run(w, x_np, g_np, steps=5, warmup=1, budget_s=25.0)
        except Exception as ex:  # noqa: BLE001
            cb = {"error": str(ex)}
        out["cpu_baseline"] = cb
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


def cache_build_times(a, dev):
    """The one-time backward-cache build (TrainingCache: symmetry probe +
    device transpose, gnn.hpp:113-196) timed cold (the run's first build,
    `transpose_ms`) and warm: median of 5 rebuilds with the workspace pool
    already grown, plus the transpose alone."""
    import torch

    from paper_2403_14853_b200 import ops
    full, tr = [], []
    for _ in range(5):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        c = ops.TrainingCache(a, True)
        c.sum_operand()
        e1.record()
        ops.transpose(a)
        e2.record()
        torch.cuda.synchronize()
        full.append(e0.elapsed_time(e1))
        tr.append(e1.elapsed_time(e2))
    return {"warm_cache_build_ms": round(float(np.median(full)), 3), "warm_transpose_ms": round(float(np.median(tr)), 3),
            "note": "TrainingCache(a) + sum_operand(): symmetry probe + CSR->CSC transpose (bit-exact); median of 5"}


def e2e_run(a, at, w, x_np, g_np, dev, plan_f, plan_b, args, ws, dist):
    """Public-API steps with host buffers: H2D(X, dC) -> spmm -> backward spmm
    -> D2H(C, dX), every step.  Copies run on their own streams with double
    buffering, so step i's compute overlaps step i+1's uploads and step i-1's
    downloads (PCIe is full duplex); the device work is the same as `value`."""
    import torch

    from paper_2403_14853_b200 import ops
    hx = torch.from_numpy(x_np).pin_memory()
    hg = torch.from_numpy(g_np).pin_memory()
    hc = torch.empty(w.n_rows, w.k).pin_memory()
    hdx = torch.empty(w.n_cols, w.k).pin_memory()
    nb = 2
    xb = [torch.empty_like(hx, device=dev) for _ in range(nb)]
    gb = [torch.empty_like(hg, device=dev) for _ in range(nb)]
    cb = [torch.empty(w.n_rows, w.k, device=dev) for _ in range(nb)]
    db = [torch.empty(w.n_cols, w.k, device=dev) for _ in range(nb)]
    comp = torch.cuda.current_stream()
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event()  # noqa: E731
    in_free = [ev() for _ in range(nb)]   # compute finished reading xb/gb[b]
    out_free = [ev() for _ in range(nb)]  # download finished reading cb/db[b]
    for e in in_free + out_free:
        e.record(comp)
    # the first upload and the last download cannot overlap: amortised over
    # up to 100 steps (~0.6 s)
    steps = max(6, min(args.steps, 100))

    def step(i):
        b = i % nb
        with torch.cuda.stream(up):
            up.wait_event(in_free[b])
            xb[b].copy_(hx, non_blocking=True)
            x_ready = ev()
            x_ready.record(up)
            gb[b].copy_(hg, non_blocking=True)
            g_ready = ev()
            g_ready.record(up)
        comp.wait_event(out_free[b])
        comp.wait_event(x_ready)
        ops.spmm_plan(a, xb[b], "sum", plan_f, cb[b])
        c_ready = ev()
        c_ready.record(comp)
        comp.wait_event(g_ready)
        ops.spmm_plan(at, gb[b], "sum", plan_b, db[b])
        in_free[b].record(comp)
        d_ready = ev()
        d_ready.record(comp)
        with torch.cuda.stream(down):
            down.wait_event(c_ready)
            hc.copy_(cb[b], non_blocking=True)
            down.wait_event(d_ready)
            hdx.copy_(db[b], non_blocking=True)
            out_free[b].record(down)

    for i in range(3):
        step(i)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    up.wait_stream(comp)
    down.wait_stream(comp)
    for i in range(steps):
        step(i)
    comp.wait_stream(down)
    comp.wait_stream(up)
    e1.record(comp)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if dist:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    flops = 2 * (2 * w.nnz * w.k) * steps * ws
    return {"value": round(flops / (ms * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
            "h2d_bytes_per_step": hx.numel() * 4 + hg.numel() * 4,
            "d2h_bytes_per_step": hc.numel() * 4 + hdx.numel() * 4,
            "ms_per_step": round(ms / steps, 4), "steps": steps,
            "note": "graph (CSR + cached CSC) resident on the device like the reference's TrainingCache; "
                    "dense inputs/outputs cross PCIe every step from/to pinned host memory on copy "
                    "streams, double-buffered so uploads/downloads overlap neighbouring steps' SpMMs"}


def run_reference_cfg2(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    w, x_np, g_np = build_workload(args.seed)
    cb = cpu_reference_run(w, x_np, g_np, steps=args.steps, warmup=args.warmup, budget_s=150.0)
    if cb is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference at build time)"}))
        return
    out = {
        "impl": "reference", "metric": METRIC, "value": round(cb["value"], 3), "unit": "GFLOP/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(cb["ms_per_step"], 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded R-MAT, BASELINE cfg2 shapes)", "config": config_of(w, {"l2": "n/a (CPU)"}),
        "cpu_baseline": {"value": round(cb["value"], 3), "unit": "GFLOP/s", "cores": cb["cores"],
                         "kind": "reference", "sample": cb["sample"], "kernel": cb["kernel"]},
        "e2e": {"value": round(cb["value"], 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


class L2Flush:
    """Between timed steps: write a 256 MiB buffer (larger than the 126 MB
    L2), then read another 256 MiB one, so the flush's own dirty lines are
    written back before the timed region starts instead of inside it (L2
    then holds clean, unrelated lines)."""

    def __init__(self, device):
        import torch
        self.w = torch.empty(256 << 20, dtype=torch.uint8, device=device)
        self.r = torch.zeros(256 << 20, dtype=torch.uint8, device=device)

    def zero_(self):  # (drop-in for the old `flush.zero_()`)
        self.w.zero_()
        self.r.max()


# ------------------------------------------------------- secondary workloads
def _events_time(fn, steps, warmup, flush=None):
    """Per-step CUDA-event times (flush outside the events), ms list."""
    import torch
    for _ in range(max(3, warmup)):
        if flush is not None:
            flush.zero_()
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(steps):
        if flush is not None:
            flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        out.append((s, e))
    torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in out]


def _base_line(args, ws, value, ms, config, extra):
    peak, src = peaks()
    line = {"metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded R-MAT, BASELINE shapes; paper datasets not available offline)",
            "config": config}
    line.update(extra)
    if "roofline" in line:
        line["roofline"].update({"peak": peak, "peak_source": src,
                                 "frac": round(line["roofline"]["achieved"] / peak, 4)})
    return line


def run_cfg1(args):
    """cfg1 (BASELINE configs[0], the reference's CPU-runnable case): one SpMM
    sum, ER 16384^2 with 16 distinct columns per row, K = 32 -- a 38 MB
    problem, so launch and memory latency dominate."""
    import torch

    from paper_2403_14853_b200 import graphs, ops
    torch.cuda.set_device(0)
    w = graphs.cfg1(args.seed)
    m, nnz, k = w.n_rows, w.nnz, w.k
    a = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
    x = torch.from_numpy(graphs.uniform(w.n_cols * k, -1.0, 1.0, args.seed, stream=12).reshape(w.n_cols, k)).cuda()
    c = torch.empty(m, k, device="cuda")
    plan = ops.Plan(a, k)
    flush = L2Flush("cuda")
    with ClockSampler(0) as clk:
        t = _events_time(lambda: ops.spmm_plan(a, x, "sum", plan, c), max(args.steps, 50), args.warmup, flush)
    # warm L2, back to back: the launches are queued behind a device-side
    # sleep so host launch overhead (~20 us through Python) is not timed
    nw = max(args.steps, 50)
    torch.cuda.synchronize()
    torch.cuda._sleep(20_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(nw):
        ops.spmm_plan(a, x, "sum", plan, c)
    e1.record()
    torch.cuda.synchronize()
    ms, ms_w = float(np.median(t)), e0.elapsed_time(e1) / nw
    by = spmm_bytes(m, nnz, k)
    cfg = {"workload": "cfg1: SpMM sum, ER 16384^2, 16 distinct uniform cols/row, vals U[-1,1], X 16384x32 U[-1,1]",
           "n_rows": m, "nnz": nnz, "K": k, "l2": "flushed between steps (256 MiB write + 256 MiB read), "
           "flush not timed; median of the steps", "plan": plan.params}
    line = _base_line(args, 1, 2 * nnz * k / ms / 1e6, ms, cfg, {
        "roofline": {"bound": "hbm", "achieved": round(by / ms / 1e6, 1), "unit": "GB/s", "traffic": None,
                     "alg_bytes_per_step": by},
        "warm_l2_ms_per_step": round(ms_w, 5), "gpu_launches": max(args.steps, 50)})
    line["steps"] = max(args.steps, 50)
    line["clocks"] = clk.summary()
    print(json.dumps(line), flush=True)


def run_cfg4(args):
    """FusedMM (sigmoid edge op, sum) + SDDMM alone on cfg4."""
    import torch

    from paper_2403_14853_b200 import graphs, ops
    torch.cuda.set_device(0)
    w = graphs.cfg4(args.seed)
    m, nnz, k = w.n_rows, w.nnz, w.k
    p = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
    x = torch.from_numpy(graphs.normal(m * k, 0, 0.1, args.seed, 41).reshape(m, k)).cuda()
    y = torch.from_numpy(graphs.normal(w.n_cols * k, 0, 0.1, args.seed, 42).reshape(w.n_cols, k)).cuda()
    out = torch.empty(m, k, device="cuda")
    flush = L2Flush("cuda")
    plan = p.plan(k, "fused")
    with ClockSampler(0) as clk:
        tf = _events_time(lambda: ops.fusedmm(p, x, y, "sigmoid_mul", "sum", out, plan=plan), args.steps, args.warmup, flush)
    ts = _events_time(lambda: ops.sddmm(p, x, y), max(5, args.steps // 4), args.warmup, flush)
    mf, msd = float(np.median(tf)), float(np.median(ts))
    fu_bytes = 8 * (m + 1) + 8 * nnz + 8 * m * k + 4 * nnz * k
    sd_bytes = 8 * (m + 1) + 8 * nnz + 4 * m * k + 4 * nnz * k + 4 * nnz
    cfg = {"workload": "cfg4: FusedMM e_ij = sigmoid(<X_i,Y_j>) a_ij, out = sum_j e_ij Y_j; R-MAT 2^20, N*32 "
                       "samples, dedup", "n_rows": m, "nnz": nnz, "K": k, "a_ij": "U[0,1]", "X,Y": "N(0,0.1)",
           "l2": "flushed between steps (256 MiB write + 256 MiB read), flush not timed", "plan": plan.params}
    line = _base_line(args, 1, 2 * nnz * k / mf / 1e6, mf, cfg, {
        "roofline": {"bound": "hbm", "achieved": round(fu_bytes / mf / 1e6, 1), "unit": "GB/s",
                     "alg_bytes_per_step": fu_bytes, **traffic_fields("cfg4", mf, peaks()[0])},
        "gflops_4nnzK": round(4 * nnz * k / mf / 1e6, 1),
        "sddmm": {"ms": round(msd, 4), "GFLOP/s": round(2 * nnz * k / msd / 1e6, 1),
                  "achieved_GBps": round(sd_bytes / msd / 1e6, 1)},
        "gpu_launches": args.steps * spmm_launches(plan, w.row_ptr)})
    line["clocks"] = clk.summary()
    print(json.dumps(line), flush=True)


def run_cfg3(args):
    """GCN layer fwd + bwd: A_hat (device normalize), SpMM(A_hat, H W) and
    A_hat^T G (symmetric: the cached operand is A_hat), dense GEMMs timed apart."""
    import torch

    from paper_2403_14853_b200 import gnn, graphs, ops
    torch.cuda.set_device(0)
    rp, ci = graphs.cfg3_graph(args.seed)
    n, k = len(rp) - 1, 256
    a = ops.CsrMatrix.from_numpy(rp, ci, np.ones(len(ci), np.float32), n)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cache = gnn.build_cache("gcn", a, True)
    e1.record()
    torch.cuda.synchronize()
    build_ms = e0.elapsed_time(e1)
    a_hat = cache.a_hat
    nnz = a_hat.nnz
    h = torch.from_numpy(graphs.normal(n * k, 0, 1, args.seed, 31).reshape(n, k)).cuda()
    lim = float(np.sqrt(6.0 / 512))
    wt = (torch.rand(k, k, generator=torch.Generator().manual_seed(args.seed)) * 2 - 1).mul(lim).cuda()
    g = torch.from_numpy(graphs.normal(n * k, 0, 1, args.seed, 32).reshape(n, k)).cuda()
    hw = h @ wt
    out = torch.empty(n, k, device="cuda")
    flush = L2Flush("cuda")
    plan = a_hat.plan(k)

    def sparse():
        ops.spmm_plan(a_hat, hw, "sum", plan, out)          # forward propagation
        cache.spmm_backward(g, "sum", out)                   # A_hat^T G (symmetric short-circuit)

    from paper_2403_14853_b200 import gnn as _gnn

    def dense():  # H W and H^T (A_hat^T G): tensor-core FP32 products (sgnn_dense_mm_f32)
        _gnn.dense_mm(h, wt)
        _gnn.dense_mm(h, out, transpose_a=True)

    with ClockSampler(0) as clk:
        tsp = _events_time(sparse, args.steps, args.warmup, flush)
    tde = _events_time(dense, max(5, args.steps // 4), args.warmup, flush)
    ms_sp, ms_de = float(np.median(tsp)), float(np.median(tde))
    by = 2 * spmm_bytes(n, nnz, k)
    cfg = {"workload": "cfg3: GCN layer fwd+bwd, A_hat = D^-1/2(A+I)D^-1/2 of R-MAT 2^20 avg-deg 50 symmetrised; "
                       "sparse = SpMM(A_hat, HW) + A_hat^T G; dense HW, H^T(A_hat^T G) (tensor-core FP32 products) timed apart",
           "n_rows": n, "nnz": nnz, "K": k, "l2": "flushed between steps (256 MiB write + 256 MiB read), flush not timed", "plan": plan.params}
    line = _base_line(args, 1, 2 * 2 * nnz * k / ms_sp / 1e6, ms_sp, cfg, {
        "roofline": {"bound": "hbm", "achieved": round(by / ms_sp / 1e6, 1), "unit": "GB/s",
                     "alg_bytes_per_step": by, **traffic_fields("cfg3", ms_sp / 2, peaks()[0])},
        "dense_ms": round(ms_de, 4), "layer_ms": round(ms_sp + ms_de, 4),
        "normalize_and_cache_ms": round(build_ms, 3), "cache_counters": cache.counters,
        "gpu_launches": args.steps * 2 * spmm_launches(plan, a_hat.to_numpy()[0])})
    line["clocks"] = clk.summary()
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    ws = int(os.environ.get("WORLD_SIZE", "0") or 0)
    if args.gpus > 1 and ws == 0:  # not under torchrun: become N ranks
        sys.exit(spawn_ranks(args.gpus, sys.argv[1:], check_gpus=not args.dry_run_dist))
    if ws and args.gpus != ws and not (args.gpus == 1 and ws == 1):
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={ws}"}), flush=True)
        sys.exit(2)
    if args.dry_run_dist:
        dry_run_dist(args)
    elif args.impl == "reference":
        if args.workload == "cfg2":
            run_reference_cfg2(args)
        elif args.workload == "cfg5":
            run_reference_cfg5(args)
        else:
            print(json.dumps({"impl": "reference", "unavailable": f"no reference arm for {args.workload}"}))
    elif args.workload == "cfg5":
        run_loopback_cfg5(args) if args.loopback else run_cfg5(args)
    elif args.workload == "cfg2":
        run_cfg2(args)
    elif args.workload == "cfg1":
        run_cfg1(args)
    elif args.workload == "cfg3":
        run_cfg3(args)
    else:
        run_cfg4(args)


if __name__ == "__main__":
    main()
