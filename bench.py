#!/usr/bin/env python
"""CALU_PRRP / LU_PRRP factorization throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Headline workload (north_star, BASELINE config 5): CALU_PRRP of U(-1,1)
n = 32768 (seed 42, 8 GiB FP64), panel b = 128, tau = 2, binary tournament
tree over P = 8 row blocks.  One step = one full factorization with the
matrix resident in HBM (a fresh device copy is restored between steps,
outside the timed region; the 8 GiB input exceeds the 126 MB L2, so no flush
is needed).  value = (2n^3/3) / t_factor in GFLOP/s, device-timed with CUDA
events on the launching stream.

  N = 1   the single-GPU driver (prrp_caluprrp: three-stream look-ahead,
          graph-captured, replayed)
  N > 1   under torchrun, one process per GPU: the distributed driver
          (dist.py / prrp_calu_dist_*): column block-cyclic layout, the
          panel owner's tournament broadcast over NCCL, every rank updating
          its own columns; value = whole-job GFLOP/s over the max-over-ranks
          time (strong scaling: the problem size is fixed)

Secondary lines in `config` (N = 1): LU_PRRP on config 2 (randn 8192,
b = 64 and 128), CALU_PRRP on config 4 (randn 16384, b = 64), and
calu_factor (the GEPP tournament baseline, n = 8192).

--impl reference times the reference algorithm's CPU implementation (the
numpy restatement in oracle/, bit-identical to the reference package on the
fixture host) on a bounded sample of the same workload, with all host cores:
the first panel of config 5 on the columns that panel's pivoting and update
reach (the first 2b columns), GFLOP/s over that sample's algorithmic flops.
"""
import argparse
import ctypes
import json
import os
import platform
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# before any CUDA context exists (see paper_1208_2451_b200/__init__.py)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

METRIC = "CALU_PRRP factorization GFLOP/s (2n^3/3), BASELINE config 5"
UNIT = "GFLOP/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--b", type=int, default=128)
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--tau", type=float, default=2.0)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--cpu-panels", type=int, default=1, help="panels per stratum of the bounded CPU sample")
    ap.add_argument("--cpu-strata", type=int, default=3, help="depths of the factorization the CPU sample covers")
    return ap.parse_args()


def dist_info():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def lu_flops(n):
    return 2.0 * n ** 3 / 3.0


def rect_lu_flops(m, w):
    """Algorithmic flops of the LU of an m x w (m >= w) matrix: m w^2 - w^3/3."""
    return m * w * w - w ** 3 / 3.0


def cpu_info():
    model = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model


def workload(args, ws):
    return {"workload": f"CALU_PRRP BASELINE config 5: U(-1,1) n={args.n} (seed {args.seed}), b={args.b}, "
                        f"tau={args.tau}, binary tournament tree P={args.P}",
            "n": args.n, "b": args.b, "P": args.P, "tau": args.tau, "matrix_bytes": args.n * args.n * 8,
            "l2": "input 8 GiB > 126 MB L2 (no flush needed); fresh device copy restored between steps",
            "parallelism": (f"column block-cyclic over {ws} GPUs (process grid 1 x {ws}), panel owner's "
                            "tournament broadcast over NCCL" if ws > 1 else "single GPU")}


# ------------------------------------------------------------------ reference arm
def cpu_sample(args, a_cols=None):
    """The oracle on a bounded, STRATIFIED sample of config 5: one panel (its
    tournament, L21, block-row finish and the update of the next panel's
    columns) at three depths of the factorization -- panel 0 on the real
    first 2b columns, and panels at 1/3 and 2/3 of the way on U(-1,1)
    stand-ins of the trailing matrix at that depth (same shape and entry
    family; the cost does not depend on the values).  Returns (seconds,
    flops, description)."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count()))
    from oracle import prrp_oracle as orc
    from paper_1208_2451_b200 import matgen
    k = max(1, args.cpu_panels)
    w = (k + 1) * args.b
    if a_cols is None:
        a_cols = matgen.gen_urand_cols(args.n, args.seed, w)
    npan = args.n // args.b
    depths = [0] if args.cpu_strata <= 1 else [round(i * npan / args.cpu_strata) for i in range(args.cpu_strata)]
    total_t, total_f, parts = 0.0, 0.0, []
    for d in depths:
        m = args.n - d * args.b
        if m < w + args.b:
            continue
        if d == 0:
            blk = np.asfortranarray(a_cols[:, :w])
        else:
            blk = np.asfortranarray(2.0 * np.random.Generator(np.random.PCG64(args.seed + d)).random((m, w)) - 1.0)
        t0 = time.perf_counter()
        orc.calu_prrp(blk, args.b, args.tau, "binary", args.P, panel_limit=k)
        dt = time.perf_counter() - t0
        fl = rect_lu_flops(m, w) - rect_lu_flops(m - k * args.b, w - k * args.b)
        total_t += dt
        total_f += fl
        parts.append(f"panel {d} ({m} rows): {dt:.1f} s")
    desc = (f"oracle.calu_prrp (numpy/OpenBLAS restatement of tournament.py:237-296), {k} panel(s) at "
            f"{len(parts)} depths of config 5 (n={args.n}, b={args.b}, P={args.P}), each restricted to the "
            f"{w} columns the panel pivots and updates [{'; '.join(parts)}]; panel 0 on the real columns, the "
            f"deeper ones on U(-1,1) stand-ins of the trailing matrix; GFLOP/s over the samples' algorithmic flops "
            f"m w^2 - w^3/3 (first {k} panels). The sample is tournament-dominated: the full factorization runs a "
            f"larger share of BLAS-2 updates (SURVEY 8(d) extrapolates ~1.5 GFLOP/s for the whole run)")
    return total_t, total_f, desc


def cpu_descr():
    return {"cores": os.cpu_count(), "cpu_model": cpu_info(),
            "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
            "openblas_coretype": os.environ.get("OPENBLAS_CORETYPE", "(unset: OpenBLAS DYNAMIC_ARCH auto-detect)")}


def run_reference(args):
    ws, rank, _ = dist_info()
    if rank != 0:
        return
    from paper_1208_2451_b200 import matgen
    a_cols = matgen.gen_urand_cols(args.n, args.seed, (max(1, args.cpu_panels) + 1) * args.b)
    times = []
    desc, flops = "", 0.0
    for i in range(args.warmup + args.steps):
        dt, flops, desc = cpu_sample(args, a_cols)
        if i >= args.warmup:
            times.append(dt)
    t = statistics.mean(times)
    value = flops / t / 1e9
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference matgen conventions: PCG64 seed 42)",
            "impl": "reference", "config": dict(workload(args, 1), sample=desc),
            "cpu_baseline": dict({"value": value, "unit": UNIT, "kind": "port", "sample": desc}, **cpu_descr()),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ device arm
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}.csv")

    def start(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def calu_call(lib, _lib, buf, n, b, tau, P, perm, timing=None):
    npc = (n + b - 1) // b
    sw = (ctypes.c_int32 * npc)()
    chg = (ctypes.c_int64 * npc)()
    st, err = _lib.PrrpStats(), _lib.PrrpErr()
    if timing is None:
        rc = lib.prrp_caluprrp(ctypes.c_void_p(buf.data_ptr()), buf.stride(0), n, n, b, float(tau), P,
                               ctypes.c_void_p(perm.data_ptr()), sw, chg, ctypes.byref(st), ctypes.byref(err),
                               _lib.stream_handle())
    else:
        rc = lib.prrp_caluprrp_timed(ctypes.c_void_p(buf.data_ptr()), buf.stride(0), n, n, b, float(tau), P,
                                     ctypes.c_void_p(perm.data_ptr()), sw, chg, ctypes.byref(st), ctypes.byref(err),
                                     ctypes.byref(timing), _lib.stream_handle())
    _lib.raise_for(rc, err, "prrp_caluprrp")
    return st, list(sw)


def timed(torch, fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1), out


def roofline_from_timing(tms, pk, what):
    """Roofline of the dominant kernel (the DMMA Schur update) from per-launch
    event spans: algorithmic flops 2 M N K summed over the launches / summed
    launch time."""
    from paper_1208_2451_b200 import _lib
    si = _lib.KCLASSES.index("schur")
    schur_ms = statistics.mean(t.ms[si] for t in tms)
    launches = statistics.mean(t.launches[si] for t in tms)
    flops = tms[0].schur_flops
    achieved = flops / (schur_ms * 1e-3) / 1e12
    breakdown = {k: round(statistics.mean(t.ms[i] for t in tms), 3) for i, k in enumerate(_lib.KCLASSES)}
    return {"bound": "tensor", "kernel": "schur_ws_kernel / schur_dmma_kernel (DMMA.8x8x4, TMA-fed)",
            "achieved": achieved, "peak": pk, "unit": "TFLOP/s", "frac": achieved / pk if pk else None,
            "peak_source": "measured live: register-resident mma.sync.m8n8k4.f64 on all SMs, 1.5 s "
                           "(prrp_b200_dmma_peak; MEASURED_PEAKS.json has no FP64 entry)",
            "achieved_def": f"{what}: sum over launches of 2*M*N*K / summed Schur launch time (CUDA events on "
                            "each launch's stream, direct enqueue)",
            "schur_flops_per_step": flops, "schur_ms_per_step": schur_ms, "schur_launches_per_step": launches,
            "step_breakdown_ms (summed spans, streams overlap)": breakdown}


def attach_traffic(roof, name):
    prof = os.path.join(ROOT, "profiles", name)
    if os.path.exists(prof):
        try:
            ps = json.load(open(prof))
            roof["traffic"] = ps.get("dram_bytes_per_launch")
            roof["traffic_note"] = ps.get("note")
        except Exception:
            roof["traffic"] = None
    else:
        roof["traffic"] = None
    return roof


def hbm_kernels():
    """ncu evidence for the HBM / latency-bound kernels of the path (north_star:
    HBM GB/s of the panel and permutation kernels), read from the committed
    summaries; the HBM peak is MEASURED_PEAKS.json's copy bandwidth."""
    peak = 6454.6
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    out = {"hbm_peak_gbs": peak}
    for key, name in (("permute_cols_kernel", "ncu_permute_cols_r02.json"),
                      ("panel_lat_kernel 128x256", "ncu_lat_128x256_r02.json"),
                      ("panel_qrcp1_kernel (config 2)", "ncu_qrcp1_c2b64_r02.json")):
        try:
            d = json.load(open(os.path.join(ROOT, "profiles", name)))
            gbs = d.get("dram_gbs")
            out[key] = {"dram_gbs": gbs, "frac_of_hbm_peak": gbs / peak if gbs else None,
                        "time_us": (d.get("time_s") or 0) * 1e6, "bound": "hbm" if key.startswith("permute") else
                        "latency (dependent pivot steps)", "source": "profiles/" + name}
        except Exception:
            continue
    return out


def run_device(args):
    import torch
    ws, rank, local = dist_info()
    torch.cuda.set_device(local)
    # PRRP_BENCH_DIST=1: the distributed driver even at N = 1 (exercises the
    # NCCL path on one GPU; the N = 1 headline uses the single-GPU driver)
    use_dist = ws > 1 or os.environ.get("PRRP_BENCH_DIST") == "1"
    if use_dist:
        import torch.distributed as dist
        if ws == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1208_2451_b200 import _lib, matgen
    from paper_1208_2451_b200 import dist as pd
    import paper_1208_2451_b200 as prrp
    lib = _lib.device_lib()
    n, b, tau, P = args.n, args.b, args.tau, args.P

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    def max_over_ranks(x):
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    pk = ctypes.c_double(0.0)
    lib.prrp_b200_dmma_peak(1500.0, ctypes.byref(pk), ctypes.byref(_lib.PrrpErr()))
    peak = pk.value

    # ---- inputs resident in HBM
    if not use_dist:
        cols = np.arange(n)
        a_loc = matgen.gen_urand(n, args.seed, order="C")
    else:
        cols = pd.local_columns(n, b, ws, rank)
        a_loc = matgen.gen_urand_colset(n, args.seed, cols)
    nl = len(cols)
    lda = max(2, nl + (nl & 1))
    pristine = torch.zeros((n, lda), dtype=torch.float64, device="cuda")
    pristine[:, :nl].copy_(torch.from_numpy(a_loc))
    work = torch.empty_like(pristine)
    perm = torch.empty(n, dtype=torch.int64, device="cuda")
    tree = prrp.binary_tree(P)

    def step():
        if not use_dist:
            return calu_call(lib, _lib, work, n, b, tau, P, perm)[0]
        return pd.caluprrp_factor_dist_device(work, n, n, b, tau, tree).stats

    for _ in range(args.warmup):
        work.copy_(pristine)
        barrier()
        timed(torch, step)
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    times = []
    for _ in range(args.steps):
        work.copy_(pristine)
        barrier()
        ms, st = timed(torch, step)
        times.append(max_over_ranks(ms))
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms_step = statistics.mean(times)
    value = lu_flops(n) / (ms_step * 1e-3) / 1e9
    growth = (st.intermediate_max / st.original_max) if not use_dist else st.growth_factor
    launches = None
    if not use_dist:
        launches = int(lib.prrp_b200_graph_kernels()) * args.steps

    extra = {"step_ms": [round(t, 2) for t in times], "growth_factor": growth}
    roofline = None
    if not use_dist:
        # per-class spans of the same factorization (direct enqueue, every launch timed)
        tms = []
        for _ in range(2):
            work.copy_(pristine)
            tm = _lib.PrrpTiming()
            calu_call(lib, _lib, work, n, b, tau, P, perm, timing=tm)
            tms.append(tm)
        roofline = attach_traffic(roofline_from_timing(tms, peak, "config 5 CALU_PRRP"), "ncu_schur_c5_r02.json")
        extra["timed_run_launches_per_step"] = int(sum(tms[-1].launches))
        extra["hbm_kernels (ncu --set full, profiles/)"] = hbm_kernels()
    del pristine, work
    torch.cuda.empty_cache()

    # ---- end to end through the public API (host buffers, H2D + D2H in the timed region)
    e2e = None
    if args.e2e_steps > 0:
        if not use_dist:
            pinned = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
            pinned.copy_(torch.from_numpy(a_loc))
            a_pin = pinned.numpy()
            et = []
            for _ in range(args.e2e_steps):
                t0 = time.perf_counter()
                f = prrp.caluprrp_factor(a_pin, b, tau, tree)
                et.append(time.perf_counter() - t0)
            del f
            e_s = statistics.mean(et)
            e2e = {"value": lu_flops(n) / e_s / 1e9, "unit": UNIT, "seconds_per_step": e_s,
                   "h2d_bytes_per_step": n * n * 8, "d2h_bytes_per_step": 2 * n * n * 8 + n * 8,
                   "timing": "wall clock around prrp.caluprrp_factor(numpy array in pinned memory) -> "
                             "BlockLUFactors (H2D, device factorization, device split, D2H of l, u, perm)"}
            del pinned, a_pin
        else:
            pinned = torch.empty((n, nl), dtype=torch.float64, pin_memory=True)
            pinned.copy_(torch.from_numpy(a_loc))
            out = torch.empty((n, nl), dtype=torch.float64, pin_memory=True)
            pout = torch.empty(n, dtype=torch.int64, pin_memory=True)
            et = []
            for _ in range(args.e2e_steps):
                barrier()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                A = torch.zeros((n, lda), dtype=torch.float64, device="cuda")
                A[:, :nl].copy_(pinned, non_blocking=True)
                f = pd.caluprrp_factor_dist_device(A, n, n, b, tau, tree)
                out.copy_(f.lu[:, :nl], non_blocking=True)
                pout.copy_(f.perm, non_blocking=True)
                torch.cuda.synchronize()
                et.append(max_over_ranks(time.perf_counter() - t0))
                del A, f
            e_s = statistics.mean(et)
            e2e = {"value": lu_flops(n) / e_s / 1e9, "unit": UNIT, "seconds_per_step": e_s,
                   "h2d_bytes_per_step": n * n * 8, "d2h_bytes_per_step": n * n * 8 + ws * n * 8,
                   "timing": "wall clock (max over ranks): every rank's columns H2D from pinned memory, "
                             "caluprrp_factor_dist_device, the packed local L\\U and perm D2H"}

    # ---- bounded CPU sample (rank 0, N = 1)
    cpu = None
    if rank == 0 and not use_dist and not args.no_cpu:
        try:
            dt, flops, desc = cpu_sample(args, np.asfortranarray(a_loc[:, :(max(1, args.cpu_panels) + 1) * b]))
            cpu = dict({"value": flops / dt / 1e9, "unit": UNIT, "kind": "port", "sample": desc}, **cpu_descr())
        except Exception as exc:  # pragma: no cover - reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {exc}"}
    del a_loc

    # ---- secondary workloads (N = 1)
    if not use_dist and not args.no_secondary:
        extra["lu_prrp_config2"] = lu_prrp_lines(lib, _lib, torch, matgen, peak, args)
        extra["calu_prrp_config4"] = calu_secondary(lib, _lib, torch, matgen, 16384, 64, "randn", args, peak)
        extra["calu_factor_gepp_n8192"] = calu_secondary(lib, _lib, torch, matgen, 8192, 64, "randn", args, peak,
                                                         gepp=True)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (U(-1,1) with the reference's matgen conventions: PCG64 seed 42, row-major fill)",
                "config": dict(workload(args, ws), **extra), "roofline": roofline, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": launches, "clocks": clk,
                "driver": "distributed (prrp_calu_dist_*, NCCL)" if use_dist else "single-GPU graph (prrp_caluprrp)",
                "fp64_peak_fraction": (value / ws / 1e3) / peak if peak else None, "fp64_peak_tflops": peak}
        print(json.dumps(line), flush=True)
    if use_dist:
        torch.distributed.destroy_process_group()


def lu_prrp_lines(lib, _lib, torch, matgen, peak, args):
    """LU_PRRP on BASELINE config 2 (randn(8192, seed 42), tau = 2), b = 64 and 128."""
    n = 8192
    a = matgen.gen_randn(n, args.seed, order="C")
    pristine = torch.from_numpy(a).cuda()
    work = torch.empty_like(pristine)
    perm = torch.empty(n, dtype=torch.int64, device="cuda")
    out = {}
    for b in (64, 128):
        def run(tm=None):
            work.copy_(pristine)
            sw = (ctypes.c_int32 * ((n + b - 1) // b))()
            st, err = _lib.PrrpStats(), _lib.PrrpErr()
            fn = lambda: lib.prrp_luprrp_timed(ctypes.c_void_p(work.data_ptr()), n, n, n, b, float(args.tau),
                                               ctypes.c_void_p(perm.data_ptr()), sw, ctypes.byref(st),
                                               ctypes.byref(err), ctypes.byref(tm) if tm is not None else None,
                                               _lib.stream_handle())
            ms, rc = timed(torch, fn)
            _lib.raise_for(rc, err, "prrp_luprrp")
            return ms, st
        for _ in range(3):
            run()
        ts = [run()[0] for _ in range(args.steps)]
        tms = []
        for _ in range(2):
            tm = _lib.PrrpTiming()
            run(tm)
            tms.append(tm)
        ms = statistics.mean(ts)
        v = lu_flops(n) / (ms * 1e-3) / 1e9
        out[f"b{b}"] = {"workload": f"LU_PRRP BASELINE config 2: randn(8192, seed {args.seed}), b={b}, tau=2",
                        "ms_per_step": ms, "value": v, "unit": UNIT, "fp64_peak_fraction": v / 1e3 / peak,
                        "step_ms": [round(t, 2) for t in ts],
                        "roofline": attach_traffic(roofline_from_timing(tms, peak, f"config 2 LU_PRRP b={b}"),
                                                   f"ncu_schur_c2b{b}_r02.json")}
    del pristine, work
    torch.cuda.empty_cache()
    return out


def calu_secondary(lib, _lib, torch, matgen, n, b, gen, args, peak, gepp=False):
    a = (matgen.gen_urand if gen == "urand" else matgen.gen_randn)(n, args.seed, order="C")
    pristine = torch.from_numpy(a).cuda()
    del a
    work = torch.empty_like(pristine)
    perm = torch.empty(n, dtype=torch.int64, device="cuda")
    ts = []
    for i in range(2 + max(2, args.steps // 2)):
        work.copy_(pristine)
        if gepp:
            chg = (ctypes.c_int64 * ((n + b - 1) // b))()
            st, err = _lib.PrrpStats(), _lib.PrrpErr()
            ms, rc = timed(torch, lambda: lib.prrp_calu(ctypes.c_void_p(work.data_ptr()), n, n, n, b, 8,
                                                        ctypes.c_void_p(perm.data_ptr()), chg, ctypes.byref(st),
                                                        ctypes.byref(err), _lib.stream_handle()))
            _lib.raise_for(rc, err, "prrp_calu")
        else:
            ms, (st, _) = timed(torch, lambda: calu_call(lib, _lib, work, n, b, args.tau, 8, perm))
        if i >= 2:
            ts.append(ms)
    del pristine, work
    torch.cuda.empty_cache()
    ms = statistics.mean(ts)
    v = lu_flops(n) / (ms * 1e-3) / 1e9
    name = "calu_factor (GEPP tournament)" if gepp else "CALU_PRRP BASELINE config 4"
    return {"workload": f"{name}: {gen}({n}, seed {args.seed}), b={b}, binary tree P=8, 1 GPU",
            "ms_per_step": ms, "value": v, "unit": UNIT, "fp64_peak_fraction": v / 1e3 / peak,
            "growth_factor": st.intermediate_max / st.original_max}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_device(args)


if __name__ == "__main__":
    main()
