#!/usr/bin/env python
"""LU_PRRP factorization throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One step = one full LU_PRRP factorization of BASELINE config 2 (randn(8192,
seed 42), panel b=64, tau=2) with the matrix already resident in HBM (a
fresh device copy is restored between steps, outside the timed region).
value = (2n^3/3) / t_factor in GFLOP/s, device-timed with CUDA events.
The 512 MiB input exceeds the 126 MB L2, so no extra flush is needed.

LU_PRRP does not shard (replicas only): under torchrun every
rank factors its own replica; value = N * F / max-over-ranks time.

--impl reference times the reference algorithm's CPU implementation (the
numpy restatement in oracle/, bit-identical to the reference package on the
fixture host) on a bounded sample of the same workload: the first panels of
the same factorization, GFLOP/s over those panels' share of 2n^3/3.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LU_PRRP factorization GFLOP/s (2n^3/3)"
UNIT = "GFLOP/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--b", type=int, default=64)
    ap.add_argument("--tau", type=float, default=2.0)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-panels", type=int, default=2, help="panels in the bounded CPU sample")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--secondary-b", type=int, default=128, help="also report this panel width (0 = off)")
    ap.add_argument("--calu-n", type=int, default=16384,
                    help="also time CALU_PRRP (BASELINE config 4: randn(n), b=64, binary tree P=8); 0 = off")
    ap.add_argument("--gcalu-n", type=int, default=8192, help="calu_factor (GEPP tournament) size (0 = off)")
    ap.add_argument("--calu5-n", type=int, default=32768,
                    help="also time CALU_PRRP (BASELINE config 5 on 1 GPU: U(-1,1), b=128, P=8); 0 = off")
    return ap.parse_args()


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def lu_flops(n):
    return 2.0 * n ** 3 / 3.0


def panel_share_flops(n, col0, bj):
    s = n - col0
    return 2.0 * (s ** 3 - (s - bj) ** 3) / 3.0


def config_dict(args, extra=None):
    d = {"workload": f"LU_PRRP BASELINE config 2: randn(n={args.n}, seed {args.seed}), b={args.b}, tau={args.tau}",
         "n": args.n, "b": args.b, "tau": args.tau, "matrix_bytes": args.n * args.n * 8,
         "l2": "input 512 MiB > 126 MB L2 (no flush needed); fresh copy restored between steps",
         "parallelism": "replicas" if int(os.environ.get("WORLD_SIZE", "1")) > 1 else "single-gpu"}
    if extra:
        d.update(extra)
    return d


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    ws, rank, _ = dist_info()
    if rank != 0:
        return
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count()))
    from oracle import prrp_oracle as orc
    a = orc.randn_matrix(args.n, args.seed)
    panels = max(1, args.cpu_panels)
    flops = sum(panel_share_flops(args.n, k * args.b, args.b) for k in range(panels))
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        orc.lu_prrp(a, args.b, args.tau, panel_limit=panels)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    t = statistics.mean(times)
    value = flops / t / 1e9
    cores = os.cpu_count()
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference matgen recipe, seed 42)",
            "impl": "reference",
            "config": config_dict(args, {"sample": f"first {panels} panels of the factorization per step"}),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"oracle.lu_prrp (numpy/OpenBLAS restatement of luprrp.py:153-201), "
                                       f"first {panels} of {args.n // args.b} panels of n={args.n}, b={args.b}; "
                                       f"GFLOP/s over their share of 2n^3/3",
                             "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS")},
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
        if os.environ.get("PRRP_BENCH_NOCLOCKS"):
            return
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


def device_run(lib, _lib, torch, pristine, work, m, n, lda, b, tau, timed=True):
    import ctypes
    work.copy_(pristine)
    perm = torch.empty(m, dtype=torch.int64, device=work.device)
    npan = (n + b - 1) // b
    swaps = (ctypes.c_int32 * npan)()
    st = _lib.PrrpStats()
    err = _lib.PrrpErr()
    tm = _lib.PrrpTiming()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    rc = lib.prrp_luprrp_timed(ctypes.c_void_p(work.data_ptr()), lda, m, n, b, float(tau),
                               ctypes.c_void_p(perm.data_ptr()), swaps, ctypes.byref(st), ctypes.byref(err),
                               ctypes.byref(tm) if timed else None, _lib.stream_handle())
    e1.record()
    e1.synchronize()
    _lib.raise_for(rc, err, "prrp_luprrp_timed")
    return e0.elapsed_time(e1), tm, st


def run_device(args):
    import torch
    ws, rank, local = dist_info()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1208_2451_b200 import _lib, matgen
    import paper_1208_2451_b200 as prrp
    lib = _lib.device_lib()

    n, b, tau = args.n, args.b, args.tau
    a_host = matgen.gen_randn(n, args.seed, order="C")          # row-major == device layout
    m = n
    lda = n + (n & 1)
    pristine = torch.empty((m, lda), dtype=torch.float64, device="cuda")
    pristine[:, :n].copy_(torch.from_numpy(a_host))
    work = torch.empty_like(pristine)

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    def max_over_ranks(x):
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        device_run(lib, _lib, torch, pristine, work, m, n, lda, b, tau)
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    times, tms = [], []
    for _ in range(args.steps):
        barrier()
        # the timed steps run the plain entry point (no per-kernel timing spans)
        ms, _, st = device_run(lib, _lib, torch, pristine, work, m, n, lda, b, tau, timed=False)
        times.append(max_over_ranks(ms))
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    # per-class breakdown and launch counts from separate instrumented runs
    for _ in range(2):
        _, tm, _ = device_run(lib, _lib, torch, pristine, work, m, n, lda, b, tau, timed=True)
        tms.append(tm)
    launches = args.steps * sum(tms[-1].launches)
    ms_step = statistics.mean(times)
    value = ws * lu_flops(n) / (ms_step * 1e-3) / 1e9
    if os.environ.get("PRRP_BENCH_STEPS"):
        print("step ms:", [round(t, 2) for t in times], file=sys.stderr, flush=True)

    # roofline of the dominant kernel (Schur update on the FP64 tensor pipe)
    schur_ms = sum(t.ms[_lib.KCLASSES.index("schur")] for t in tms) / len(tms)
    schur_launch = sum(t.launches[_lib.KCLASSES.index("schur")] for t in tms) / len(tms)
    schur_flops = tms[0].schur_flops
    import ctypes
    pk = ctypes.c_double(0.0)
    err = _lib.PrrpErr()
    lib.prrp_b200_dmma_peak(1500.0, ctypes.byref(pk), ctypes.byref(err))
    achieved = schur_flops / (schur_ms * 1e-3) / 1e12
    traffic, traffic_note = None, None
    prof = os.path.join(ROOT, "profiles", "ncu_schur_r01.json")
    if os.path.exists(prof):
        try:
            ps = json.load(open(prof))
            traffic = ps.get("dram_bytes_per_launch")
            traffic_note = (f"dram read+write of {ps.get('reference_launch')} from {ps.get('report')}; "
                            f"algorithmic bytes of that launch {ps.get('algorithmic_bytes_reference_launch')}")
        except Exception:
            traffic = None
    breakdown = {k: round(sum(t.ms[i] for t in tms) / len(tms), 4) for i, k in enumerate(_lib.KCLASSES)}
    roofline = {"bound": "tensor", "kernel": "schur_dmma_kernel (DMMA.8x8x4, TMA-fed)", "achieved": achieved,
                "peak": pk.value, "unit": "TFLOP/s", "frac": achieved / pk.value if pk.value else None,
                "traffic": traffic, "traffic_note": traffic_note,
                "peak_source": "measured live: register-resident mma.sync.m8n8k4.f64 loop on all SMs, 1.5 s "
                               "(MEASURED_PEAKS.json has no FP64 entry)",
                "achieved_def": "sum over panels of 2*M*N*b / summed schur_dmma_kernel event time per step",
                "launches_per_step": schur_launch, "schur_ms_per_step": schur_ms,
                "step_breakdown_ms": breakdown}

    extra = {}
    # secondary panel width (b=128) on the same matrix
    if args.secondary_b and args.secondary_b != b:
        for _ in range(2):
            device_run(lib, _lib, torch, pristine, work, m, n, lda, args.secondary_b, tau)
        t2 = []
        for _ in range(max(2, args.steps // 2)):
            barrier()
            ms, _, _ = device_run(lib, _lib, torch, pristine, work, m, n, lda, args.secondary_b, tau, timed=False)
            t2.append(max_over_ranks(ms))
        ms2 = statistics.mean(t2)
        extra["secondary"] = {"b": args.secondary_b, "ms_per_step": ms2,
                              "value": ws * lu_flops(n) / (ms2 * 1e-3) / 1e9, "unit": UNIT}

    def calu_line(cn, cb, gen, label, reps=2, gepp=False):
        """CALU_PRRP (binary tree, P = 8) on a device-resident matrix; the first two
        calls capture and upload the factorization's CUDA graph (untimed)."""
        import ctypes
        ca = (matgen.gen_urand if gen == "urand" else matgen.gen_randn)(cn, args.seed, order="C")
        cld = cn + (cn & 1)
        cprist = torch.empty((cn, cld), dtype=torch.float64, device="cuda")
        cprist[:, :cn].copy_(torch.from_numpy(ca))
        del ca
        cwork = torch.empty_like(cprist)
        cperm = torch.empty(cn, dtype=torch.int64, device="cuda")
        npc = (cn + cb - 1) // cb
        ct = []
        for i in range(2 + reps):
            cwork.copy_(cprist)
            sw = (ctypes.c_int32 * npc)()
            chg = (ctypes.c_int64 * npc)()
            cst, cerr = _lib.PrrpStats(), _lib.PrrpErr()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if gepp:   # calu_factor: the GEPP-tournament baseline (one stream, no graph)
                rc = lib.prrp_calu(ctypes.c_void_p(cwork.data_ptr()), cld, cn, cn, cb, 8,
                                   ctypes.c_void_p(cperm.data_ptr()), chg, ctypes.byref(cst), ctypes.byref(cerr),
                                   _lib.stream_handle())
            else:
                rc = lib.prrp_caluprrp(ctypes.c_void_p(cwork.data_ptr()), cld, cn, cn, cb, float(tau), 8,
                                       ctypes.c_void_p(cperm.data_ptr()), sw, chg, ctypes.byref(cst),
                                       ctypes.byref(cerr), _lib.stream_handle())
            e1.record()
            e1.synchronize()
            _lib.raise_for(rc, cerr, "prrp_caluprrp")
            if i >= 2:
                ct.append(e0.elapsed_time(e1))
        cms = statistics.mean(ct)
        del cprist, cwork, cperm
        torch.cuda.empty_cache()
        v = lu_flops(cn) / (cms * 1e-3) / 1e9
        if gepp:
            return {"workload": f"calu_factor (GEPP tournament) {label}({cn}, seed {args.seed}), b={cb}, binary "
                                "tree P=8, 1 GPU", "ms_per_step": cms, "value": v, "unit": UNIT,
                    "growth_factor": cst.intermediate_max / cst.original_max,
                    "timing": f"CUDA events around prrp_calu, mean of {reps} steps after 2 untimed"}
        return {"workload": f"CALU_PRRP {label}({cn}, seed {args.seed}), b={cb}, tau={tau}, binary tree P=8, 1 GPU",
                "ms_per_step": cms, "value": v, "unit": UNIT,
                "fp64_peak_fraction": (v / 1e3) / pk.value if pk.value else None,
                "swaps": int(sum(sw)), "growth_factor": cst.intermediate_max / cst.original_max,
                "timing": f"CUDA events around prrp_caluprrp, mean of {reps} steps after 2 untimed "
                          "(graph capture + upload)"}

    # BASELINE config 4: CALU_PRRP, randn(16384, seed 42), b = 64, binary tournament tree over P = 8
    if args.calu_n and rank == 0:
        extra["calu_config4"] = calu_line(args.calu_n, 64, "randn", "randn")
    # BASELINE config 5 on one GPU: CALU_PRRP, U(-1,1) n = 32768 (8 GiB), b = 128, P = 8
    if args.calu5_n and rank == 0:
        extra["calu_config5"] = calu_line(args.calu5_n, 128, "urand", "urand")
    # the reference's tournament-pivoted GEPP baseline (tournament.py:299-359), SURVEY 8(f)
    if args.gcalu_n and rank == 0:
        extra["calu_factor"] = calu_line(args.gcalu_n, 64, "randn", "randn", gepp=True)

    # end to end through the public API: host input in pinned memory -> device -> factors on host
    e2e = None
    if args.e2e_steps > 0:
        pinned = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        pinned.copy_(torch.from_numpy(a_host))
        a_pin = pinned.numpy()
        prrp.luprrp_factor(a_pin, b, tau)
        et = []
        for _ in range(args.e2e_steps):
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f = prrp.luprrp_factor(a_pin, b, tau)
            et.append(max_over_ranks(time.perf_counter() - t0))
        e_s = statistics.mean(et)
        e2e = {"value": ws * lu_flops(n) / e_s / 1e9, "unit": UNIT, "seconds_per_step": e_s,
               "h2d_bytes_per_step": n * n * 8, "d2h_bytes_per_step": 2 * n * n * 8 + m * 8,
               "timing": "wall clock around prrp.luprrp_factor(numpy in pinned memory) -> BlockLUFactors "
                         "(H2D, device factorization, device split of L/U, D2H of l, u, perm)"}
        extra["growth_factor"] = f.stats.growth_factor

    cpu = None
    if rank == 0 and not args.no_cpu:
        try:
            os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count()))
            from oracle import prrp_oracle as orc
            panels = max(1, args.cpu_panels)
            a_f = np.asfortranarray(a_host)
            t0 = time.perf_counter()
            orc.lu_prrp(a_f, b, tau, panel_limit=panels)
            dt = time.perf_counter() - t0
            flops = sum(panel_share_flops(n, k * b, b) for k in range(panels))
            cpu = {"value": flops / dt / 1e9, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                   "sample": f"oracle.lu_prrp (numpy/OpenBLAS restatement of the reference), first {panels} "
                             f"of {n // b} panels of n={n}, b={b} ({dt:.1f} s); GFLOP/s over their share of 2n^3/3"}
        except Exception as exc:  # pragma: no cover - reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {exc}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference matgen recipe: PCG64 seed 42, "
                                                           "Box-Muller normals, row-major fill)",
                "config": config_dict(args, extra), "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk,
                "fp64_peak_fraction": (value / ws / 1e3) / pk.value if pk.value else None}
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_device(args)


if __name__ == "__main__":
    main()
