"""Benchmark: ANOVA-Laplacian matvecs/s (fp64) + CG denoise solve time.

One *step* is one batched fused system matvec  y_r = v_r + a_r (eta v_r -
Gamma v_r)  for the config-4 alpha sweep (16 right-hand sides sharing every
Gamma application; BASELINE.json configs[4], 4096x4096, N = 16,777,216,
3 windows of 3 features, M = 32, m = 4, fp64).  Matvecs count per right-hand
side.  Inputs are device resident (2.1 GB of vectors + 9.7 GB of node tables,
far larger than the 126 MB L2, so no explicit flush).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--impl reference` times the reference's CPU algorithm (the C+numpy port in
oracle/, all host threads) on a bounded sample of the same workload and
prints the same metric.  Under torchrun (N > 1) the pixels are sharded over
the ranks (strong scaling): each rank spreads its slice, one NCCL allreduce
sums the per-window support-box grids, every rank convolves redundantly and
gathers its own pixels; CG scalars are allreduced.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "ANOVA-Laplacian matvecs/s (fp64)"
UNIT = "matvec/s"
SAMPLE_NODES = 1 << 20        # CPU baseline: pixels [0, 2^20) of the config


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--nrhs", type=int, default=0, help="0: config default")
    ap.add_argument("--no-cg", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=32,
                    help="batches streamed through the pipelined host API (its one-batch "
                         "fill and drain amortised over them); 0: --steps")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------------------
# CPU baseline (reference algorithm, C + numpy port, all host threads)
# --------------------------------------------------------------------------

def cpu_sample(cfg_name, steps=2, warmup=1):
    from oracle.cpu_port import CpuPort
    import synth

    feats, wins, _ = synth.make_problem(cfg_name)
    n_full = feats.shape[0]
    ns = min(SAMPLE_NODES, n_full)
    sub = np.ascontiguousarray(feats[:ns])
    port = CpuPort(sub, wins, synth.SIGMA, n_expansion=synth.N_EXPANSION,
                   cutoff=synth.CUTOFF, oversampling=synth.OVERSAMPLING)
    eta = port.degree()
    mu = synth.ALPHA_SCALE / float(eta.mean())
    v = synth.random_vector(ns)
    for _ in range(warmup):
        port.system_apply(v, 1.0, mu)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        port.system_apply(v, 1.0, mu)
        times.append(time.perf_counter() - t0)
    scale = ns / n_full
    best = min(times)
    return {
        "value": scale / best,
        "unit": UNIT,
        "cores": port.nthreads,
        "kind": "port",
        "sample": (f"{cfg_name} pixels [0,{ns}) of {n_full} (all {len(wins)} "
                   f"windows, M=32, m=4), one single-RHS ShiftedSystem.apply "
                   f"per step on {port.nthreads} host threads (C restatement of "
                   f"_kernels.py spread/gather + numpy pocketfft), best of "
                   f"{steps} after {warmup} warm-up; scaled by {ns}/{n_full}"),
        "sample_seconds": best,
        "host_cpus": os.cpu_count(),
        "times_s": times,
        "n_full": n_full,
        "windows": [len(w) for w in wins],
    }


REF_SAMPLE_NODES = 1 << 17   # the real reference (numba, one thread): pixels [0, 2^17)


def reference_numba_sample(cfg_name, nodes=REF_SAMPLE_NODES):
    """The UNMODIFIED reference package (baseline/_ref, installed offline from
    /root/reference/pkg) timed through its own public API: one
    ShiftedSystem.apply (linops.py:48-50 -> kernel.py:79-93) per step, after a
    warm-up that JIT-compiles its numba loops, on the first `nodes` pixels
    of the config, scaled by nodes/N.  Its loops are serial
    (_kernels.py:48,91), so this is one host thread.  As in the golden
    generator only `_build_plans` is overridden, to pass the
    BASELINE NFFT parameters that kernel.py:74 otherwise hard-codes."""
    ref_dir = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "nldenoise")):
        return {"value": None, "sample": "unavailable: baseline/_ref not installed"}
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    try:
        from nldenoise import kernel as rk
        from nldenoise import linops as rl
        from nldenoise import transform as rt
    except Exception as exc:  # numba / scipy missing on this host
        return {"value": None, "sample": f"unavailable: {exc}"}
    import synth

    class Pinned(rk.AnovaOperator):
        def _build_plans(self, sigbar):
            plans = []
            for w in self.windows:
                pts = np.ascontiguousarray(self.features[:, w])
                plan = rt.FastsumPlan.build(pts, sigbar, n_expansion=synth.N_EXPANSION,
                                            cutoff=synth.CUTOFF,
                                            oversampling=synth.OVERSAMPLING)
                plans.append((pts, plan, plan.tables_for(pts)))
            return plans

    feats, wins, _ = synth.make_problem(cfg_name)
    n_full = feats.shape[0]
    ns = min(nodes, n_full)
    op = Pinned(np.ascontiguousarray(feats[:ns]), wins, synth.SIGMA)
    eta = op.degree()                      # builds the plans + JIT warm-up
    system = rl.ShiftedSystem(op, 1.0, synth.ALPHA_SCALE / float(eta.mean()))
    v = synth.random_vector(ns)
    t0 = time.perf_counter()
    system.apply(v)
    best = time.perf_counter() - t0
    return {"value": (ns / n_full) / best, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample_seconds": best,
            "sample": (f"UNMODIFIED reference nldenoise (baseline/_ref, numba, one thread): "
                       f"ShiftedSystem.apply on pixels [0,{ns}) of {n_full} of {cfg_name} "
                       f"(M=32, m=4 via the _build_plans override), one timed call after "
                       f"a JIT warm-up, scaled by {ns}/{n_full}")}


def workload_config(cfg_name, nrhs, n_global, n_rank, windows, world, kernels, setup_s=None):
    """The `config` object of both arms' lines (same workload, same keys)."""
    import synth
    cfg = {"workload": (f"{cfg_name}: batched fused system matvec "
                        f"y = v + a_k(eta v - Gamma v), {nrhs} rhs "
                        "(pixel-major batch)"),
           "n_nodes": int(n_global), "nodes_per_rank": int(n_rank),
           "windows": list(windows), "nrhs": int(nrhs),
           "bandwidth": synth.N_EXPANSION, "cutoff": synth.CUTOFF, "grid": 64,
           "parallelism": (f"pixel-sharded x{world} (grid allreduce over NCCL)"
                           if world > 1 else "single"),
           "l2": "inputs larger than L2 (no flush)", "kernels": kernels}
    if setup_s is not None:
        cfg["setup_s"] = setup_s
    return cfg


def run_reference(args, world, rank):
    if rank != 0:
        return
    res = cpu_sample(args.config, steps=max(1, args.steps), warmup=max(0, args.warmup))
    try:
        numba_ref = reference_numba_sample(args.config)
    except Exception as exc:  # the extra sample must not sink the line
        numba_ref = {"value": None, "sample": f"failed: {exc}"}
    line = {
        "metric": METRIC, "value": res["value"], "unit": UNIT,
        "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * res["sample_seconds"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        # the same workload and metric as our arm (matvecs per rhs): the
        # sample (cpu_baseline.sample) is a bounded slice of it, scaled
        "config": workload_config(args.config, args.nrhs or 16, res["n_full"],
                                  res["n_full"], res["windows"], world,
                                  "reference algorithm on the host CPU: C restatement of "
                                  "_kernels.py spread/gather + numpy FFT (all host threads)"),
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind",
                                             "sample")},
        "host_cpus": os.cpu_count(),
        "reference_numba": numba_ref,
        "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# clocks during the timed region
# --------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,"
              "clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [],
                    "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------

def ncu_traffic(kernel_tag):
    """dram bytes per launch of the dominant kernel from the committed
    `ncu --set full` summary (profiles/ncu_summary.json), if present."""
    path = os.path.join(REPO, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            data = json.load(fh)
        ent = data.get("kernels", {}).get(kernel_tag)
        return None if ent is None else ent.get("dram_bytes_per_product")
    except (OSError, ValueError):
        return None


def run_ours(args, world, rank, local):
    import torch

    import paper_2407_06834_b200 as nld
    from paper_2407_06834_b200 import _lib, sharding
    import synth

    # NLD_TEST_SHARED_GPU=1: every rank on cuda:0 over gloo -- a functional
    # check of the sharded flow on a one-GPU box (numbers meaningless)
    shared = os.environ.get("NLD_TEST_SHARED_GPU", "") not in ("", "0")
    local = 0 if shared else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        pg = dist
    cfg = synth.CONFIGS[args.config]
    # the throughput line is the 16-rhs batch at every config (c4: its alpha
    # sweep; c2/c3: 16 right-hand sides sharing each product); the config's
    # own solve (c2: one image, c3: three channels) is timed in `cg`
    nrhs = args.nrhs or 16
    feats, wins, f_img = synth.make_problem(args.config)
    n_global = feats.shape[0]
    # pixel sharding (strong scaling): this rank's pixels, partitioned by
    # window-0 stencil-cell ownership (sharding.partition)
    ix = sharding.partition(feats, wins, world)[rank] if world > 1 else np.arange(n_global)
    feats = np.ascontiguousarray(feats[ix])
    f_img = np.ascontiguousarray(f_img[ix])
    n = len(ix)
    feat_t = torch.from_numpy(feats).to(dev)
    t_setup = time.perf_counter()
    op = nld.AnovaOperator(feat_t, wins, synth.SIGMA,
                           n_expansion=synth.N_EXPANSION, cutoff=synth.CUTOFF,
                           oversampling=synth.OVERSAMPLING)
    if world > 1:
        sharding.attach(op, sharding.TorchComm(device=dev), rank, n_global)
    eta = op.degree_device()
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    eta_sum = eta.sum()
    if pg:
        pg.all_reduce(eta_sum)
    mean_eta = float(eta_sum) / n_global
    alphas = (synth.alpha_sweep(mean_eta, nrhs) if cfg.n_alpha > 1
              else np.full(nrhs, synth.ALPHA_SCALE / mean_eta))
    coef = np.stack([np.ones(nrhs), alphas], axis=1).ravel()
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    # batch in the kernels' native pixel-major layout (n, nrhs): rhs fastest
    V = torch.randn((n, nrhs), dtype=torch.float64, device=dev, generator=gen)
    Y = torch.empty_like(V)
    stream = torch.cuda.current_stream(dev)

    def step():
        op.apply_device(V, _lib.APPLY_SYSTEM, nrhs, coef, out=Y, pixel_major=True)

    # fp64 FMA peak on this GPU (roofline denominator)
    import ctypes
    tf, pms = ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.lib.nld_probe_fp64(1 << 16, 0, ctypes.byref(tf), ctypes.byref(pms),
                                       ctypes.c_void_p(stream.cuda_stream)))
    dfma_peak = tf.value
    _lib.check(_lib.lib.nld_probe_dmma(1 << 13, 0, ctypes.byref(tf), ctypes.byref(pms),
                                       ctypes.c_void_p(stream.cuda_stream)))
    dmma_peak = tf.value
    fp64_peak = max(dfma_peak, dmma_peak)
    _lib.check(_lib.lib.nld_probe_imma(1 << 14, 0, ctypes.byref(tf), ctypes.byref(pms),
                                       ctypes.c_void_p(stream.cuda_stream)))
    imma_peak = tf.value
    # the library runs 16k-rhs batches of 3-D, m = 4 windows on the
    # integer-sliced tcgen05 kernels (nld_ozaki.cu) unless NLD_OZAKI=0
    sliced = (nrhs % 16 == 0 and synth.CUTOFF == 4
              and os.environ.get("NLD_OZAKI", "1") != "0")

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    op.set_timing(True)
    stage = {"spread_ms": 0.0, "assemble_ms": 0.0, "conv_ms": 0.0,
             "gather_ms": 0.0, "epilogue_ms": 0.0}
    launches = 0
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
            st = op.stats()
            for k in stage:
                stage[k] += st[k]
            launches += st["launches"]
        ev1.record(stream)
        torch.cuda.synchronize()
    if pg:
        pg.barrier()
    op.set_timing(False)
    elapsed_ms = ev0.elapsed_time(ev1)
    if pg:
        t = torch.tensor([elapsed_ms], device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_step = elapsed_ms / max(args.steps, 1)
    # every step is nrhs matvecs of the whole (global) operator
    value = nrhs * args.steps / (elapsed_ms * 1e-3)

    # e2e through the public API: pinned host inputs -> device -> result back,
    # every step; AnovaOperator.apply_pipelined overlaps the PCIe copies of
    # neighbouring steps with the kernels (3 streams, double buffering)
    e2e_steps = max(1, args.e2e_steps or args.steps)
    Vh = torch.empty((n, nrhs), dtype=torch.float64, pin_memory=True)
    Vh.copy_(V.cpu())
    Yh = [torch.empty((n, nrhs), dtype=torch.float64, pin_memory=True) for _ in range(2)]
    del V, Y
    torch.cuda.synchronize()
    op.apply_pipelined(_lib.APPLY_SYSTEM, [Vh], [Yh[0]], nrhs, coef,
                       pixel_major=True)   # warm-up
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    op.apply_pipelined(_lib.APPLY_SYSTEM, [Vh] * e2e_steps,
                       [Yh[k & 1] for k in range(e2e_steps)], nrhs, coef,
                       pixel_major=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if pg:
        t = torch.tensor([e2e_ms], device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_val = nrhs * e2e_steps / (e2e_ms * 1e-3)
    del Vh, Yh

    # roofline of the dominant kernel (stage timings are CUDA events on the
    # launching stream, summed over the timed region)
    info = [op.window_info(w) for w in range(len(wins))]
    sum_d = sum(i["dim"] for i in info)
    flops_pt = sum(2 * (2 * synth.CUTOFF) ** i["dim"] for i in info)  # FMA=2
    dominant = "gather" if stage["gather_ms"] >= stage["spread_ms"] else "spread"
    dom_ms = stage[dominant + "_ms"] / max(args.steps, 1)
    # minimal algorithmic bytes of one launch: raw coordinates
    # (8 B per window dimension) + one fp64 vector per right-hand side
    alg_bytes = n * (8 * sum_d + 8 * nrhs)
    alg_flops = n * nrhs * flops_pt
    hbm_peak = 6458.4
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            hbm_peak = float(json.load(fh)["hbm_gbs"])
        peak_src = "MEASURED_PEAKS.json"
    except (OSError, ValueError, KeyError):
        peak_src = "fallback"
    achieved = alg_bytes / (dom_ms * 1e-3) / 1e9
    alg_tflops = alg_flops / (dom_ms * 1e-3) / 1e12
    hbm = {"achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
           "frac": achieved / hbm_peak, "peak_source": f"{peak_src} hbm_gbs",
           "bytes_model": ("minimal (SURVEY §8d): N*(8*sum_l d_l + 8*nrhs) "
                           "per launch -- not the binding roofline")}
    share = {k[:-3]: v / max(elapsed_ms, 1e-9) for k, v in stage.items()}
    if sliced:
        # int8 UMMA work actually issued: per 32 nodes and 16 rhs, 6 digit
        # rows p against (6 - p) stacked 64-wide digit slices, K = 32 (spread)
        # and the same volume for the gather (2 K steps x (6 - p) 32-node
        # slices) -> 1344 * 128 * 32 * 2 ops per 32 nodes
        n3 = sum(1 for i in info if i["dim"] == 3)
        ops = n * (nrhs // 16) * (1344 * 128 * 32 * 2 // 32) * n3
        tag = "k_gather_nm" if dominant == "gather" else "k_spread_ozp"
        tops = ops / (dom_ms * 1e-3) / 1e12
        roofline = {
            "bound": "tensor", "achieved": tops, "peak": imma_peak, "unit": "TOPS (int8)",
            "frac": tops / imma_peak,
            "traffic": ncu_traffic(tag),
            "traffic_unit": "dram bytes per product (all window launches, ncu, committed profile)",
            "kernel": tag, "kernel_ms": dom_ms,
            "peak_source": (f"int8 tcgen05 UMMA probe measured in this run (M=128 N=256 K=32, "
                            f"one CTA per SM): {imma_peak:.0f} TOPS"),
            "ops_model": ("int8 MMA ops issued per product: N*(nrhs/16)*344064 per 3-D window "
                          "(6x6 digit slices, diagonals t<=5) / the kernel's event-timed stage"),
            "fp64_equivalent": {
                "achieved": alg_tflops, "unit": "TFLOP/s",
                "dmma_peak": fp64_peak, "frac_of_dmma_peak": alg_tflops / fp64_peak,
                "flops_model": "N*nrhs*sum_l 2*(2m)^d_l (the fp64 algorithm's flops)"},
            "hbm": hbm, "stage_share": share,
        }
    else:
        tag = "k_gather_mma" if dominant == "gather" else "k_spread_mma"
        roofline = {
            # fp64 tensor path (DMMA): bound by fp64 throughput; MEASURED_PEAKS.json has
            # no fp64 figure, so the peak is measured here, in this run, on this GPU
            "bound": "tensor", "achieved": alg_tflops, "peak": fp64_peak,
            "unit": "TFLOP/s", "frac": alg_tflops / fp64_peak,
            "traffic": ncu_traffic(tag),
            "traffic_unit": "dram bytes per product (all window launches, ncu, committed profile)",
            "kernel": tag, "kernel_ms": dom_ms,
            "peak_source": (f"fp64 measured in this run: DMMA m8n8k4 probe {dmma_peak:.2f}, "
                            f"DFMA probe {dfma_peak:.2f} TFLOP/s (shared execution "
                            "resources; max taken)"),
            "flops_model": ("N*nrhs*sum_l 2*(2m)^d_l per product (all window launches of the "
                            "kernel, FMA = 2 flop) / the kernel's event-timed stage"),
            "hbm": hbm, "stage_share": share,
        }

    # single-rhs product throughput (the reference's own bench-op times one
    # ShiftedSystem.apply(v), cli.py:347-357): fp64 DMMA kernels at nrhs = 1
    single = None
    if cfg.n_alpha == 1 and not args.no_cg:
        v1 = torch.randn(n, dtype=torch.float64, device=dev, generator=gen)
        y1 = torch.empty_like(v1)
        c1v = coef[:2].copy()
        for _ in range(2):
            op.apply_device(v1, _lib.APPLY_SYSTEM, 1, c1v, out=y1, pixel_major=True)
        if pg:
            pg.barrier()
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(args.steps):
            op.apply_device(v1, _lib.APPLY_SYSTEM, 1, c1v, out=y1, pixel_major=True)
        s1.record(stream)
        torch.cuda.synchronize()
        sms = s0.elapsed_time(s1) / max(args.steps, 1)
        if pg:
            t = torch.tensor([sms], device=dev)
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            sms = float(t.item())
        single = {"value": 1e3 / sms, "unit": UNIT, "ms_per_matvec": sms,
                  "kernels": "fp64 DMMA spread/gather (nrhs = 1)"}
        del v1, y1

    # CG denoise solve (deflated Jacobi, tol 1e-6): c4 the 16-alpha sweep,
    # c2 the image, c3 its three channels as right-hand sides (alpha =
    # 10 / mean eta)
    cg = None
    if not args.no_cg:
        if cfg.n_alpha > 1:
            f = torch.from_numpy(np.ascontiguousarray(f_img[:, 0])).to(dev)
            cg_alpha = alphas
        else:
            f = torch.from_numpy(np.ascontiguousarray(f_img.T)).to(dev)
            if f.shape[0] == 1:
                f = f[0]
            cg_alpha = synth.ALPHA_SCALE / mean_eta
        # warm-up solve (2 iterations): the operator's persistent CG vectors
        # and scratch are allocated once, as for a user solving many images
        nld.deflated_solve_batched(op, f, 1.0, cg_alpha, prec="jacobi", tol=synth.CG_TOL,
                                   maxit=2)
        torch.cuda.synchronize()
        c0 = torch.cuda.Event(enable_timing=True)
        c1 = torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        res = nld.deflated_solve_batched(op, f, 1.0, cg_alpha, prec="jacobi",
                                         tol=synth.CG_TOL, maxit=200)
        c1.record(stream)
        torch.cuda.synchronize()
        its = [r.iterations for r in res]
        cg = {"solve_ms": c0.elapsed_time(c1), "nrhs": len(res),
              "rhs": ("16 alphas log-spaced over [1,100]/mean eta" if cfg.n_alpha > 1
                      else f"{cfg.channels} channel(s), alpha = 10/mean eta"),
              "iterations": its, "converged": all(r.converged for r in res),
              "relres_max": max(r.relative_residual for r in res),
              "tol": synth.CG_TOL, "prec": "jacobi (deflated)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_sample(args.config)
            cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as exc:  # the baseline must not sink the bench line
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                   "sample": f"unavailable: {exc}"}
    if cg is not None and cpu is not None and cpu.get("value"):
        nmv = sum(cg["iterations"]) + 2 * cg["nrhs"]
        cg["cpu_extrapolated_s"] = nmv / cpu["value"]
        cg["cpu_extrapolation"] = ("reference matvecs (iterations + 2 per alpha) "
                                   "x sampled CPU matvec time")

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(
                args.config, nrhs, n_global, n, [len(w) for w in wins], world,
                ("integer-sliced tcgen05 spread/gather (exact s8 x s8 -> s32 digit products, "
                 "fp64 combine)" if sliced else "fp64 DMMA spread/gather"), t_setup),
            "roofline": roofline, "cpu_baseline": cpu, "host_cpus": os.cpu_count(),
            "e2e": {"value": e2e_val, "unit": UNIT,
                    "h2d_bytes_per_step": int(nrhs * n_global * 8),
                    "d2h_bytes_per_step": int(nrhs * n_global * 8),
                    "steps": e2e_steps,
                    "api": "AnovaOperator.apply_pipelined (pinned host batches; H2D of batch "
                           "k+1, product of k, D2H of k-1 overlapped on three streams)"},
            "single_rhs": single,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "cg": cg,
        }
        print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
