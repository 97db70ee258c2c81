#!/usr/bin/env python
"""NeuRLP-PDE batched fwd+bwd solve throughput on B200 (BASELINE.json metric).

metric: PDE solves/s (fwd+bwd) at 64^2 x 32 grid, batch 32 (config C4, NS vorticity).
One step = mpde_build_hierarchy + mpde_solve_fwd + mpde_solve_bwd over the batch (every
row of SURVEY.md §8(a)) + the batch sum of grad_c and, for N > 1 GPUs, its NCCL
all-reduce (§8(e)).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config C4|C5|C2|C3]

--config C4 (default): weak scaling, every rank solves its own batch of 32 C4 PDEs.
--config C5: BASELINE configs[4], (t,x,y) = (64,128,128), global batch 256 sharded
             256/N over the ranks (strong scaling).
--config C2 / C3: the 1D Burgers (101x256, batch 64) / 2D reaction-diffusion (32^3,
             16 solves) workloads per rank (weak scaling).
With --gpus N > 1 and no WORLD_SIZE in the environment the script re-launches itself
under torch.distributed.run with N ranks (one per GPU, NCCL).

--impl reference times the fp64 CPU oracle (oracle/, the correctness reference; no
other reference implementation exists) on a bounded sample of the same workload.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}

def _baseline_metric():
    """BASELINE.json's metric string, verbatim (the driver matches the line against it)."""
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as f:
            return json.load(f)["metric"]
    except (OSError, KeyError, ValueError):
        return "PDE solves/s (fwd+bwd) at 64\u00b2\u00d732 grid, batch 32; HBM GB/s vs peak"


METRIC = _baseline_metric()
UNIT = "PDE solves/s (fwd+bwd)"
# algorithmic bytes per point of S pass 2 (k_schur_s_*), per epilogue kind: x 4 + h 4 +
# cf[7] 28 (sigma alpha, u~ 2D) read + the epilogue's vector traffic
EPI_NAMES = ["store", "dot", "lanczos", "resid", "smooth", "smooth_last", "post0"]
EPI_BYTES = [40, 40, 44, 44, 60, 52, 60]
# S pass 1 (k_schur_h_*): x 4 + cf[8] 32 (sigma alpha, 1/sigma, u~) read + h 4 written
SCHUR_G_BYTES = 40
# level-0 V-cycle applies (epilogues resid, smooth, smooth_last, post0) read the coefficients
# as bf16 when mpde_options.cf_bf16 = 1: pass 2 reads 7 of them (saves 14 B/pt), pass 1
# reads 8 (saves 16 B/pt)
BF16_EPIS = (3, 4, 5, 6)
BF16_SAVED_PASS2 = 14
BF16_SAVED_PASS1 = 16

OPT_OVERRIDES = {}  # --opt name=value (mpde_options fields; experiments only)

WORKLOADS = {
    "C4": "C4: 2D Navier-Stokes vorticity, (t,x,y)=(32,64,64), batch 32 per GPU, fwd+bwd incl. "
          "hierarchy build",
    "C5": "C5: 2D NS-vorticity scaling sweep, (t,x,y)=(64,128,128), global batch 256 sharded over "
          "the GPUs, fwd+bwd incl. hierarchy build",
    "C2": "C2: 1D Burgers template, (t,x)=(101,256), batch 64 per GPU, fwd+bwd incl. build",
    "C3": "C3: 2D lambda-omega reaction-diffusion, (t,x,y)=(32,32,32), 8 samples x 2 fields = 16 "
          "solves per GPU, fwd+bwd incl. build",
}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk, "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, gpu_index: int, path: str):
        self.path = path
        self.proc = None
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-i", str(gpu_index), "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return None
        sm = sorted(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------------ oracle sample
# The oracle as it stands solves a 3D PDE with its converging method, t-slab block-Jacobi PCG
# (oracle.solve_normal(method="slab"): SuperLU factorisation of every 2-plane slab block of the
# equilibrated normal matrix, then PCG).  Full C4 runs (tools/make_golden.py, the golden
# references) needed 475 iterations forward and 625 backward; those counts come from the
# committed sidecars tests/golden/c4_pde*.json.  A bounded sample measures, per process on one
# host core, the assembly, the normal matrix, ONE slab block's factorisation and a few block
# solves and normal-matrix products; the full fwd+bwd cost is then
#   t_asm + 2 * (n_blocks * t_factor + iters * (t_matvec + n_blocks * t_blocksolve))
SLAB_PLANES = 2


def _oracle_sample(args):
    cfg_name, idx, reps = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import numpy as np
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    import synth
    from oracle import Problem, assemble
    cfg = synth.CONFIGS[cfg_name]
    c, b, om = synth.make_pde(cfg_name, idx)
    M = c.shape[0]
    pr = Problem(cfg.shape, cfg.h)
    t0 = time.perf_counter()
    A, d, _ = assemble(pr, c.reshape(M, -1).astype(np.float32), b.reshape(-1).astype(np.float32),
                       om.reshape(-1).astype(np.float32))
    N = (A.T @ A).tocsr()
    s = 1.0 / np.sqrt(N.diagonal())
    Ns = (sp.diags(s) @ N @ sp.diags(s)).tocsr()
    t_asm = time.perf_counter() - t0
    P = pr.P
    pl = P // cfg.shape[0]
    blk = np.concatenate([m * P + np.arange(0, SLAB_PLANES * pl) for m in range(M)])
    t1 = time.perf_counter()
    lu = spla.splu(Ns[blk][:, blk].tocsc())
    t_fac = time.perf_counter() - t1
    r = np.random.default_rng(idx).normal(size=blk.size)
    t2 = time.perf_counter()
    for _ in range(reps):
        lu.solve(r)
    t_bs = (time.perf_counter() - t2) / reps
    x = np.random.default_rng(idx + 1).normal(size=N.shape[0])
    t3 = time.perf_counter()
    for _ in range(reps):
        Ns @ x
    t_mv = (time.perf_counter() - t3) / reps
    return t_asm, t_fac, t_bs, t_mv


def _oracle_iters():
    """Slab-PCG iterations of the converged C4 oracle solves (tests/golden sidecars)."""
    its = []
    for i in (0, 31):
        try:
            with open(os.path.join(ROOT, "tests", "golden", f"c4_pde{i}.json")) as f:
                j = json.load(f)
            its.append((j["fwd"]["iters"], j["bwd"]["iters"]))
        except Exception:
            pass
    if not its:
        return 475, 625
    return (sum(a for a, _ in its) / len(its), sum(b for _, b in its) / len(its))


def oracle_workers():
    """All host cores, bounded by memory (one C4 normal matrix + one slab factor ~3 GB)."""
    n = os.cpu_count() or 1
    try:
        import psutil
        n = max(1, min(n, int(psutil.virtual_memory().available / 3.5e9)))
    except Exception:
        pass
    return n


def cpu_oracle_baseline(reps=3, workers=None):
    import multiprocessing as mp
    n = workers or oracle_workers()
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(n) as pool:
        res = pool.map(_oracle_sample, [("C4", i, reps) for i in range(n)])
    wall = time.perf_counter() - t0
    i_f, i_b = _oracle_iters()
    mean = lambda k: sum(r[k] for r in res) / len(res)
    t_asm, t_fac, t_bs, t_mv = mean(0), mean(1), mean(2), mean(3)
    nblk = synth_c4_planes() // SLAB_PLANES
    per_dir = lambda it: nblk * t_fac + it * (t_mv + nblk * t_bs)
    est = t_asm + per_dir(i_f) + per_dir(i_b)  # seconds per fwd+bwd solve on one core
    return {"value": n / est, "unit": UNIT, "cores": n, "kind": "oracle",
            "host_cpus": os.cpu_count(), "cpu_model": cpu_model(),
            "sample": (f"{n} C4 PDEs (32x64x64, NS vorticity) on {n} processes x 1 thread "
                       f"({os.cpu_count()} host CPUs, {cpu_model()}): the oracle's assembly + normal "
                       f"matrix ({t_asm:.1f} s), one {SLAB_PLANES}-plane slab block's SuperLU "
                       f"factorisation ({t_fac:.1f} s), {reps} block solves ({1e3 * t_bs:.0f} ms each) and "
                       f"{reps} normal-matrix products ({1e3 * t_mv:.0f} ms each); scaled to {nblk} blocks "
                       f"and the {i_f:.0f} fwd + {i_b:.0f} bwd slab-PCG iterations of the converged "
                       f"C4 oracle runs (tests/golden/c4_pde*.json): {est / 60:.1f} min per fwd+bwd "
                       f"solve per core; {wall:.1f}s wall")}, wall


def synth_c4_planes():
    import synth
    return synth.CONFIGS["C4"].shape[0]


# ------------------------------------------------------------------------------ ours
class Workload:
    """Device-resident inputs of one rank: `nsets` input sets of `B` PDEs (alternated so that
    consecutive steps do not reuse L2-resident inputs), plus outputs and per-step stats."""

    def __init__(self, cfg_name, B, start, dev, nsets=2, distinct=None):
        import numpy as np
        import torch
        import synth
        from paper_2502_18377_b200 import mpde
        self.cfg = synth.CONFIGS[cfg_name]
        self.name = cfg_name
        self.B = B
        D = len(self.cfg.shape)
        self.M, self.P = 1 + 2 * D, int(np.prod(self.cfg.shape))
        self.prob = mpde.make_problem(self.cfg.shape, self.cfg.h, B)
        self.opts = mpde.mpde_default_options(**OPT_OVERRIDES)
        self.ws = torch.empty(mpde.mpde_workspace_bytes(self.prob, self.opts), dtype=torch.uint8,
                              device=dev)
        self.sets = []
        nd = B if distinct is None else min(B, distinct)
        self.distinct = nd
        for k in range(nsets):
            s0 = start + k * B
            bt = synth.make_batch(cfg_name, nd, start=s0)
            g = synth.make_g(cfg_name, nd, start=s0)
            reps = (B + nd - 1) // nd
            tile = lambda x: np.ascontiguousarray(np.concatenate([x] * reps, axis=0)[:B])
            arrs = (tile(bt["c"]), tile(bt["b"]), tile(bt["omega"]), tile(g))
            self.sets.append({"c": torch.from_numpy(arrs[0]).to(dev),
                              "b": torch.from_numpy(arrs[1]).to(dev),
                              "om": torch.from_numpy(arrs[2]).to(dev),
                              "g": torch.from_numpy(arrs[3]).to(dev), "np": arrs})
        M, P = self.M, self.P
        self.z = torch.empty((B, M, P), dtype=torch.float32, device=dev)
        self.gc = torch.empty_like(self.z)
        self.gb = torch.empty((B, P), dtype=torch.float32, device=dev)
        self.gw = torch.empty_like(self.gb)
        self.gsum = torch.empty((M, P), dtype=torch.float32, device=dev)
        self.dev = dev

    def input_bytes(self):
        return 4 * (2 * self.B * self.M * self.P + 2 * self.B * self.P)


def make_step(W, stream, opts=None, ws=None):
    from paper_2502_18377_b200 import mpde
    from paper_2502_18377_b200.parallel import allreduce_coeff_grad
    opts = W.opts if opts is None else opts
    ws = W.ws if ws is None else ws

    def step(i, sf=None, sb=None):
        s = W.sets[i % len(W.sets)]
        h = mpde.mpde_build_hierarchy(W.prob, opts, s["c"], ws, stream)
        mpde.mpde_solve_fwd(h, s["b"], s["om"], W.z, sf, stream)
        mpde.mpde_solve_bwd(h, s["b"], W.z, s["g"], W.gc, W.gb, W.gw, None, sb, stream)
        mpde.mpde_batch_sum(W.gc, W.gsum, stream)
        allreduce_coeff_grad(W.gsum)  # NCCL over NVLink: shared-coefficient gradient (§8(e))
        mpde.mpde_destroy_hierarchy(h)
    return step


def timed(step, steps, warmup, stream, world, dev, stats=None):
    """W untimed warm-up steps, then exactly K steps between barrier + synchronize, CUDA
    events on the launching stream; returns the max over ranks of the elapsed ms."""
    import torch
    import torch.distributed as dist
    from paper_2502_18377_b200.parallel import max_over_ranks
    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for i in range(steps):
        if stats is None:
            step(warmup + i)
        else:
            step(warmup + i, stats[0][i], stats[1][i])
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    return max_over_ranks(ev0.elapsed_time(ev1), device=dev)


def summarize_stats(stats, dev):
    """Per-PDE iterations and failures over EVERY timed step (not only the last one)."""
    import torch
    from paper_2502_18377_b200.parallel import max_over_ranks
    sf = torch.stack(stats[0]).cpu()  # [K][B][5]
    sb = torch.stack(stats[1]).cpu()
    out = {"fwd_mean": float(sf[..., 0].float().mean()), "bwd_mean": float(sb[..., 0].float().mean()),
           "fwd_max": int(max_over_ranks(int(sf[..., 0].max()), device=dev)),
           "bwd_max": int(max_over_ranks(int(sb[..., 0].max()), device=dev)),
           "not_converged": int(max_over_ranks(int((sf[..., 2] != 0).sum() + (sb[..., 2] != 0).sum()),
                                               device=dev))}
    return out


def profile_roofline(W, step, stream):
    """One profiled step (outside the timed region): per-class CUDA-event times of every
    library launch on the solver's stream, and the roofline of the dominant kernel class
    (achieved = algorithmic bytes of the points it processed / its summed event time)."""
    from paper_2502_18377_b200 import mpde
    import torch
    mpde.mpde_profile_begin()
    step(0)
    prof, pts = mpde.mpde_profile_end()
    torch.cuda.synchronize()
    tot_ms = sum(v[0] for v in prof.values())
    bf = W.opts.cf_bf16
    so_ms, so_n = prof["schur_out_l0"]
    so_bytes = sum(p * (bb - (BF16_SAVED_PASS2 if bf and e in BF16_EPIS else 0))
                   for e, (p, bb) in enumerate(zip(pts[9:16], EPI_BYTES)))
    sg_ms, sg_n = prof["schur_g_l0"]
    sg_bytes = pts[7] * SCHUR_G_BYTES - (BF16_SAVED_PASS1 if bf else 0) * sum(pts[9 + e] for e in BF16_EPIS)
    sc_ms, sc_n = prof["schur_out"]
    sc_bytes = sum(p * bb for p, bb in zip(pts[:7], EPI_BYTES))
    peaks, peak_kind = load_peaks()
    peak = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    gbs = lambda b, ms: b / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(W.name, {}).get("schur_out_bytes_per_launch")
        except Exception:
            traffic = None
    achieved = gbs(so_bytes, so_ms)
    roof = {"bound": "hbm", "kernel": "S pass 2 on level 0 (k_schur_s_*, fused PCG/smoother epilogues)",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak if peak else None,
            "traffic": traffic, "peak_kind": peak_kind, "launches": so_n,
            "bytes_per_launch": so_bytes / max(so_n, 1),
            "avg_launch_us": 1e3 * so_ms / max(so_n, 1),
            "share_of_step": so_ms / tot_ms if tot_ms else None}
    extra = {"schur_g_l0": {"achieved_gbs": gbs(sg_bytes, sg_ms),
                            "frac": gbs(sg_bytes, sg_ms) / peak if peak else None,
                            "share_of_step": sg_ms / tot_ms if tot_ms else None},
             "schur_out_coarse": {"achieved_gbs": gbs(sc_bytes, sc_ms), "launches": sc_n,
                                  "share_of_step": sc_ms / tot_ms if tot_ms else None}}
    kernels = {k: {"ms": v[0], "launches": v[1]} for k, v in prof.items()}
    return roof, extra, kernels


def sub_step(cfg_name, a, stream, world, rank, dev):
    """Value + roofline of another BASELINE workload on this rank (weak scaling)."""
    import torch
    import synth
    cfg = synth.CONFIGS[cfg_name]
    W = Workload(cfg_name, cfg.batch, rank * 2 * cfg.batch, dev)
    step = make_step(W, stream)
    K = max(1, a.steps)
    st = ([torch.zeros((W.B, 5), dtype=torch.int32, device=dev) for _ in range(K)],
          [torch.zeros((W.B, 5), dtype=torch.int32, device=dev) for _ in range(K)])
    ms = timed(step, K, a.warmup, stream, world, dev, st)
    roof, extra, _ = profile_roofline(W, step, stream)
    out = {"value": world * W.B * K / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / K,
           "workload": WORKLOADS[cfg_name], "iters": summarize_stats(st, dev),
           "roofline": {k: roof[k] for k in ("achieved", "peak", "frac", "share_of_step", "avg_launch_us")}}
    out.update(extra)
    del W
    return out


def run_ours(a):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_2502_18377_b200 import mpde
    from paper_2502_18377_b200.parallel import allreduce_coeff_grad, max_over_ranks, shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    cfg_name = a.config
    cfg = synth.CONFIGS[cfg_name]
    if cfg_name == "C5":  # strong scaling: the global batch is sharded over the ranks
        start, B = shard(cfg.batch, rank, world)
        scaling = "strong"
        nsets, distinct = 1, 32
    else:
        B, start = cfg.batch, rank * 2 * cfg.batch
        scaling = "weak"
        nsets, distinct = 2, None
    stream = torch.cuda.current_stream()
    W = Workload(cfg_name, B, start, dev, nsets=nsets, distinct=distinct)
    M, P = W.M, W.P
    in_mb = W.input_bytes() / 1e6
    step = make_step(W, stream)
    K = a.steps
    stats = ([torch.zeros((B, 5), dtype=torch.int32, device=dev) for _ in range(K)],
             [torch.zeros((B, 5), dtype=torch.int32, device=dev) for _ in range(K)])

    # warm-up, then the timed region (clocks sampled during it)
    for i in range(a.warmup):
        step(i)
    torch.cuda.synchronize()
    clocks = ClockSampler(local, os.path.join(ROOT, "gpurun_out", f"clocks_r{rank}.csv")) \
        if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else ClockSampler(local, f"/tmp/clocks_{rank}.csv")
    time.sleep(0.5)
    l0 = mpde.mpde_launch_count()
    ms = timed(step, K, 0, stream, world, dev, stats)
    launches = mpde.mpde_launch_count() - l0
    clk = clocks.stop()
    iters = summarize_stats(stats, dev)
    total_B = cfg.batch if cfg_name == "C5" else world * B
    value = total_B * K / (ms / 1e3)
    if iters["not_converged"] > 0:
        print(f"bench: {iters['not_converged']} PDE solves did not converge in the timed steps",
              file=sys.stderr)

    # ---- phase breakdown (outside the timed region): build / fwd / bwd, CUDA events ----
    phases = {}
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    s0 = W.sets[0]
    torch.cuda.synchronize()
    evs[0].record(stream)
    hh = mpde.mpde_build_hierarchy(W.prob, W.opts, s0["c"], W.ws, stream)
    evs[1].record(stream)
    mpde.mpde_solve_fwd(hh, s0["b"], s0["om"], W.z, None, stream)
    evs[2].record(stream)
    mpde.mpde_solve_bwd(hh, s0["b"], W.z, s0["g"], W.gc, W.gb, W.gw, None, None, stream)
    evs[3].record(stream)
    mpde.mpde_batch_sum(W.gc, W.gsum, stream)
    evs[4].record(stream)
    torch.cuda.synchronize()
    mpde.mpde_destroy_hierarchy(hh)
    for k, name in enumerate(["build", "fwd", "bwd", "grad_sum"]):
        phases[name] = evs[k].elapsed_time(evs[k + 1])

    roof, extra, kernels = profile_roofline(W, step, stream)

    # ---- end to end through the host-buffer C-ABI call ------------------------------
    e2e = None
    if not a.no_e2e:
        need = 2 * W.input_bytes() * len(W.sets)
        try:
            import psutil
            avail = psutil.virtual_memory().available
        except Exception:
            avail = None
        if avail is not None and need > 0.5 * avail:
            e2e = {"value": None, "unit": UNIT,
                   "skipped": f"pinned host buffers ({need / 1e9:.1f} GB) exceed half the available "
                              f"host memory ({avail / 1e9:.1f} GB)"}
        else:
            host = []
            for s in W.sets:
                host.append(tuple(torch.from_numpy(x).pin_memory() for x in s["np"]))
            z_h = torch.empty((B, M, P), dtype=torch.float32).pin_memory()
            gc_h = torch.empty_like(z_h).pin_memory()
            gb_h = torch.empty((B, P), dtype=torch.float32).pin_memory()
            gw_h = torch.empty_like(gb_h).pin_memory()
            stg = torch.empty(mpde.mpde_host_staging_bytes(W.prob), dtype=torch.uint8, device=dev)

            def e2e_step(i):
                c_h, b_h, om_h, g_h = host[i % len(host)]
                mpde.mpde_fwd_bwd_host(W.prob, W.opts, c_h, b_h, om_h, g_h, z_h, gc_h, gb_h, gw_h,
                                       stg, W.ws, stream)

            e2e_step(0)
            ke = max(1, min(K, 5))
            te_ms = timed(e2e_step, ke, 0, stream, world, dev)
            h2d = 4 * (2 * B * M * P + 2 * B * P)
            d2h = 4 * (2 * B * M * P + 2 * B * P)
            e2e = {"value": total_B * ke / (te_ms / 1e3), "unit": UNIT,
                   "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                   "api": "mpde_fwd_bwd_host (pinned host buffers; H2D of c, b, omega, g_z and D2H of "
                          "z, grad_c, grad_b, grad_omega inside the timed region)"}
            del stg, host

    subs = {}
    if cfg_name == "C4":
        # ---- the paper's discovery step: polynomial template -> solve -> dl/dtheta -> all-reduce
        if not a.no_template:
            from paper_2502_18377_b200.parallel import allreduce_theta_grad
            tm = mpde.make_template(2, 1)
            theta = torch.from_numpy(synth.ns_template_theta()).to(dev)
            feats = [torch.from_numpy(np.ascontiguousarray(s["np"][0][:, [3, 5]])).to(dev) for s in W.sets]
            ct = torch.empty((B, M, P), dtype=torch.float32, device=dev)
            bt_ = torch.empty((B, P), dtype=torch.float32, device=dev)
            gth = torch.empty_like(theta)
            tws = torch.empty(mpde.mpde_template_workspace_bytes(W.prob, tm), dtype=torch.uint8, device=dev)

            def tstep_fn(i, sf=None, sb=None):
                s = W.sets[i % 2]
                mpde.mpde_template_coeff(W.prob, tm, theta, feats[i % 2], ct, bt_, stream)
                h = mpde.mpde_build_hierarchy(W.prob, W.opts, ct, W.ws, stream)
                mpde.mpde_solve_fwd(h, bt_, s["om"], W.z, None, stream)
                mpde.mpde_solve_bwd(h, bt_, W.z, s["g"], W.gc, W.gb, W.gw, None, None, stream)
                mpde.mpde_template_grad(W.prob, tm, theta, feats[i % 2], W.gc, W.gb, gth, None, tws, stream)
                allreduce_theta_grad(gth)  # NCCL: the shared-parameter gradient (a few hundred bytes)
                mpde.mpde_destroy_hierarchy(h)

            tms = timed(tstep_fn, K, a.warmup, stream, world, dev)
            subs["template_step"] = {
                "value": world * B * K / (tms / 1e3), "unit": UNIT, "ms_per_step": tms / K,
                "workload": "C4 as a discovery step: degree-1 template in (U1, U2) (P:552) -> "
                            "build -> fwd -> bwd -> dl/dtheta -> all-reduce of [8][3] fp32",
                "allreduce_bytes": gth.numel() * 4}
            del ct, bt_, tws

        # ---- §8(f) N1: the same C4 step with FGMRES(30) instead of PCG (the paper's Krylov method)
        if not a.no_fgmres:
            fopts = mpde.mpde_default_options(krylov=1)
            fws = torch.empty(mpde.mpde_workspace_bytes(W.prob, fopts), dtype=torch.uint8, device=dev)
            fstep = make_step(W, stream, fopts, fws)
            fst = ([torch.zeros((B, 5), dtype=torch.int32, device=dev) for _ in range(K)],
                   [torch.zeros((B, 5), dtype=torch.int32, device=dev) for _ in range(K)])
            fms = timed(fstep, K, a.warmup, stream, world, dev, fst)
            subs["fgmres_step"] = {
                "value": world * B * K / (fms / 1e3), "unit": UNIT, "ms_per_step": fms / K,
                "workload": "C4 step (build -> fwd -> bwd -> grad_c all-reduce) with FGMRES(30) "
                            "+ the same V-cycle (krylov=1) instead of PCG",
                "iters": summarize_stats(fst, dev)}
            del fws

        # ---- §8(f) N3: the dense path (levels_max = 1: exact S^-1) on C1-sized 1D problems ----
        if not a.no_dense:
            c1 = synth.CONFIGS["C1"]
            DB = 2048
            d1 = synth.make_batch("C1")
            g1 = synth.make_g("C1")
            rep = lambda x: torch.from_numpy(np.repeat(x, DB, axis=0)).to(dev)
            dc, db_, dom, dg = rep(d1["c"]), rep(d1["b"]), rep(d1["omega"]), rep(g1)
            dprob = mpde.make_problem(c1.shape, c1.h, DB)
            dopts = mpde.mpde_default_options(levels_max=1)
            dws = torch.empty(mpde.mpde_workspace_bytes(dprob, dopts), dtype=torch.uint8, device=dev)
            dz, dgc = torch.empty_like(dc), torch.empty_like(dc)
            dgb, dgw = torch.empty_like(db_), torch.empty_like(db_)
            dsf = torch.zeros((DB, 5), dtype=torch.int32, device=dev)

            def dstep_fn(i, sf=None, sb=None):
                h = mpde.mpde_build_hierarchy(dprob, dopts, dc, dws, stream)
                mpde.mpde_solve_fwd(h, db_, dom, dz, dsf, stream)
                mpde.mpde_solve_bwd(h, db_, dz, dg, dgc, dgb, dgw, None, None, stream)
                mpde.mpde_destroy_hierarchy(h)

            dms = timed(dstep_fn, K, a.warmup, stream, world, dev)
            dst = dsf.cpu()
            subs["dense_step"] = {
                "value": world * DB * K / (dms / 1e3), "unit": UNIT, "ms_per_step": dms / K,
                "workload": f"C1 heat 16x16 replicated to batch {DB} per GPU, dense path "
                            "(levels_max=1: probed S, fp64 Gauss-Jordan inverse, GEMV PCG)",
                "fwd_iters_max": int(dst[:, 0].max()), "ws_bytes": int(dws.numel())}
            del dws

        # ---- the other BASELINE workloads as sub-steps (C2 1D Burgers, C3 2D RD) ----------
        if not a.no_subconfigs:
            del W
            torch.cuda.empty_cache()
            for cn in ("C2", "C3"):
                subs[f"{cn.lower()}_step"] = sub_step(cn, a, stream, world, rank, dev)

    if rank == 0:
        cpu = None
        if world == 1 and not a.no_cpu and cfg_name == "C4":
            cpu, _ = cpu_oracle_baseline()
        data = f"synthetic (seeded {cfg.kind} coefficient fields, synth.gen {cfg_name})"
        if cfg_name == "C5":
            data += f"; {min(B, 32)} distinct PDEs per rank tiled to the shard of {B}"
        line = {
            "metric": METRIC,
            "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": a.warmup, "ms_per_step": ms / K, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f32 (fp64 refinement/condensation)",
            "data": data,
            "config": {"workload": WORKLOADS[cfg_name], "option_overrides": OPT_OVERRIDES or None,
                       "global_batch": total_B, "grid": list(cfg.shape),
                       "parallelism": f"dp{world} (batch-sharded PDEs, NCCL all-reduce of grad_c)",
                       "l2": (f"inputs larger than L2 ({nsets} input set(s) of {in_mb:.0f} MB, "
                              "alternated between steps)")},
            "roofline": roof,
            "kernels": kernels,
            "phases_ms": phases,
            "iters": iters,
            "gpu_launches": launches,
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        line.update(extra)
        line.update(subs)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------------ reference
def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    t0 = time.perf_counter()
    vals = []
    cpu = None
    for _ in range(a.steps):
        cpu, wall = cpu_oracle_baseline()
        vals.append(cpu["value"])
    el = time.perf_counter() - t0
    v = sum(vals) / len(vals)
    line = {"impl": "reference", "metric": METRIC,
            "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 * el / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS["C4"]},
            "cpu_baseline": cpu,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=["C4", "C5", "C2", "C3"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-template", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-fgmres", action="store_true")
    ap.add_argument("--no-subconfigs", action="store_true")
    ap.add_argument("--opt", action="append", default=[],
                    help="override an mpde_options field, e.g. --opt poll_every=4 (experiments)")
    a = ap.parse_args()
    for kv in a.opt:
        k, v = kv.split("=", 1)
        OPT_OVERRIDES[k] = float(v) if ("." in v or "e" in v.lower()) else int(v)
    env_world = os.environ.get("WORLD_SIZE")
    if a.impl == "ours" and a.gpus > 1 and env_world is None:
        # one process per GPU: re-launch under torch.distributed.run (NCCL, 127.0.0.1)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1",
               f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if a.impl == "ours" and env_world is not None and int(env_world) != a.gpus:
        print(f"bench: --gpus {a.gpus} but WORLD_SIZE={env_world}", file=sys.stderr)
        sys.exit(2)
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
