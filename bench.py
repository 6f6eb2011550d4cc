#!/usr/bin/env python3
"""Headline benchmark: mixed-precision DIRK time steps on a 3D heat grid.

Metric (BASELINE.json): RK time-steps/s & DOF-updates/s for the 3D heat
mixed DIRK at 256^3 (configs[1]).  `value` = DOF-updates/s of the whole job
(n^3 x steps / s, summed over ranks); `steps_per_s` rides along.

Workload (one "step" = one Stepper::step, stepper.cpp:149-206):
  heat 256^3, 4s3pB = Grant's 4-stage 3rd-order mixed DIRK (four fp32
  implicit stage solves by CG + the reference's FastDiag preconditioner,
  fp64 explicit couplings, fp64 state), tau = 0.01, tol = 1e-3 (the fp32
  attainable floor at 256^3 is 1.8e-4 relative, SURVEY.md §0 finding 4),
  max_iter 40, state resident in HBM.  (midpoint1, the 2-stage member, is
  not usable for long fp32 runs at this size: its explicit corrector
  amplifies fp32 stage rounding by ~(tau |K|)^2/2 = 3e7 per step and the run
  diverges after ~20 steps — the paper's divergence caveat.)

Arms
  default           this repo's CUDA path (libmprk_b200.so, FAST numerics)
  --impl reference  the reference's own CPU implementation (oracle/_ref, the
                    unmodified reference sources, OpenMP on all host cores),
                    same workload, bounded sample of steps.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
Multi-GPU (--gpus N > 1, under torch.distributed.run, one rank per GPU):
configs[2] — ONE 512^3 grid slab-decomposed across the N GPUs (rank r owns
k-planes [r 512/N, (r+1) 512/N)), ghost planes exchanged with the
k-neighbours before every stencil, FastDiag transposed k-slab <-> j-slab by
an all-to-all around its contraction along k, Krylov dots summed across
ranks — all over NCCL (libmprk_b200's own communicator; torch.distributed
only broadcasts the NCCL id and takes the max-over-ranks time).  Fixed total
work as N grows ("scaling": "strong"); at N = 8 each GPU holds 512*512*64 =
256^3 DOF, the N = 1 line's per-GPU size.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RK time-steps/s & DOF-updates/s, 3D heat 256³–512³ mixed DIRK; SpMV HBM GB/s"
N_GRID = 256
N_SPLIT = 512  # configs[2]: the grid split across N > 1 GPUs
METHOD = "4s3pB"
TAU = 0.01
TOL = 1e-3
PREC = "f32"
MAX_ITER = 40


def grid_for_world(n_gpus: int, split: bool = False) -> int:
    return N_SPLIT if (n_gpus > 1 or split) else N_GRID


def workload_config(n_gpus: int, split: bool = False) -> dict:
    n = grid_for_world(n_gpus, split)
    split = split or n_gpus > 1
    return {
        "workload": f"heat {n}^3, {METHOD} (4-stage mixed DIRK: fp32 implicit CG + FastDiag, "
                    f"fp64 explicit couplings/state), tau={TAU}, tol={TOL}"
                    + (f", k-slab decomposed over {n_gpus} GPU(s) (NCCL)" if split else ""),
        "n": n, "dof": n ** 3, "dof_per_gpu": n ** 3 // n_gpus, "method": METHOD, "implicit_precision": PREC,
        "preconditioner": "fastdiag", "tau": TAU, "tol": TOL, "max_iter": MAX_ITER,
        "state": "resident in HBM (f64)",
        "l2": "no flush: one step streams >= 3.5 GB per GPU through HBM (state slab alone 134 MB > 126 MB L2)",
        "parallelism": (f"slab{n_gpus} (k-planes; halo + all-to-all + dot allreduce)" if split else "single"),
    }


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------------
# clocks sampling during the timed region
# ---------------------------------------------------------------------------------
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: an NVML
    poll every 2 ms on a side thread (nvidia-smi -lms cannot start inside a
    sub-second timed region)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self.err = None
        self.run = False
        self.t = None

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001 - reported in the JSON line
            self.err = f"nvml unavailable: {e}"
            return
        self.run = True
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()
        time.sleep(0.005)

    def _poll(self):
        nv = self.nv
        while self.run:
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, rs))
            except Exception as e:  # noqa: BLE001
                self.err = str(e)
                return
            time.sleep(0.002)

    def stop(self) -> dict:
        if self.t is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "not sampled"], "samples": 0}
        self.run = False
        self.t.join(timeout=2)
        reasons = sorted(nm for nm, bit in self.REASONS.items() if any(rs & bit for _, rs in self.samples))
        sm = [s for s, _ in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(self.smax),
                "reasons": reasons, "samples": len(sm), "source": "NVML every 2 ms during the timed region"}


# ---------------------------------------------------------------------------------
# CPU reference (oracle/_ref: the reference sources compiled unmodified)
# ---------------------------------------------------------------------------------
def reference_steps(n: int, steps_wanted: int, budget_s: float, threads: int):
    """Time the reference's own Stepper::step on this host; returns
    (seconds per step list, threads, sample description)."""
    from oracle.oracle import Reference, ensure_built, have_reference

    ensure_built(ref=True)
    if not have_reference():
        return None
    R = Reference()
    R.set_threads(threads)
    tab = R.tableau(METHOD)
    st = R.stepper(0, n, tab, TAU, TOL, PREC, MAX_ITER)
    u, *_ = R.make_problem(0, n)
    times = []
    t_start = time.perf_counter()
    while len(times) < steps_wanted:
        t0 = time.perf_counter()
        st.step(u)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start + times[-1] > budget_s:
            break
    return times


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    # warm-up: at most one step (the CPU needs none for steady state; it only
    # faults in the 2 GB working set), then a bounded sample of timed steps
    budget = float(os.environ.get("MPRKB_REF_BUDGET_S", "150"))
    t0 = time.perf_counter()
    warm = reference_steps(N_GRID, min(args.warmup, 1), budget / 3, threads) if args.warmup else []
    if warm is None:
        emit({"impl": "reference", "unavailable": "oracle/_ref/libmprk_ref.so not built"})
        return 0
    times = reference_steps(N_GRID, args.steps, budget, threads)
    per_step = sum(times) / len(times)
    value = N_GRID ** 3 / per_step
    sample = (f"{len(times)} of {args.steps} requested steps of the same workload "
              f"(+{len(warm)} warm-up), wall clock, {threads} OpenMP threads")
    if world > 1:
        # one 512^3 reference step takes minutes on the host (FastDiag is
        # 12 n flop/DOF, 16x the 256^3 cost): the sample is the 256^3 step,
        # whose DOF-updates/s bounds the 512^3 rate from above
        sample = (f"{len(times)} step(s) of heat {N_GRID}^3 {METHOD} on {threads} OpenMP threads "
                  f"(upper bound on the reference's {N_SPLIT}^3 DOF-updates/s; no multi-node/GPU path "
                  f"exists in the reference)")
    line = {
        "metric": METRIC, "value": value, "unit": "DOF-updates/s", "n_gpus": args.gpus, "steps": len(times),
        "warmup": len(warm), "ms_per_step": per_step * 1e3, "steps_per_s": 1.0 / per_step,
        "higher_is_better": True, "scaling": "weak" if world == 1 else "strong", "vs_baseline": None,
        "dtype": "f32/f64", "data": "synthetic",
        "config": workload_config(world), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "DOF-updates/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "DOF-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t0,
    }
    emit(line)
    return 0


# ---------------------------------------------------------------------------------
# the CUDA arm
# ---------------------------------------------------------------------------------
def load_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu
    capture (profiles/ncu_summary.json), if present."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("dominant_kernel_dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def measure_contraction(mp, torch, stream_ptr, reps=20):
    """Average duration of one FastDiag tensor-contraction launch (the
    dominant kernel), timed with CUDA events on the launching stream."""
    n = N_GRID
    P = mp.Operator.fastdiag_stage(0, "heat", n, TAU, 0.5, "fast")
    x = torch.randn(n ** 3, dtype=torch.float32, device="cuda")
    s = torch.cuda.ExternalStream(stream_ptr) if stream_ptr else torch.cuda.current_stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            P.apply(x)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            P.apply(x)
        b.record(s)
        b.synchronize()
    ms_apply = a.elapsed_time(b) / reps
    return ms_apply / 6.0  # six contraction launches per apply (diag fused)


def run_cuda_arm(args):
    import torch

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    import paper_2412_16638_b200 as mp

    split = world > 1 or args.split
    n = N_SPLIT if split else N_GRID
    m = n ** 3  # DOF of the whole (possibly split) grid
    tab = mp.builtin(METHOD)
    comm = None
    if split:
        # libmprk_b200's own NCCL communicator; torch.distributed only ships the
        # id (--split at one GPU: a 1-rank communicator, every exchange path
        # against itself — the N > 1 code path on a single-GPU box)
        mp.set_device(local)
        if world > 1:
            obj = [mp.Comm.nccl_unique_id() if rank == 0 else None]
            torch.distributed.broadcast_object_list(obj, src=0)
            uid = obj[0]
        else:
            uid = mp.Comm.nccl_unique_id()
        comm = mp.Comm.nccl(rank, world, uid)
    st = mp.Stepper("heat", n, tab, TAU, TOL, PREC, MAX_ITER, comm=comm)
    stream = torch.cuda.ExternalStream(st.stream)
    u = torch.from_numpy(st.initial_state()).cuda()  # this rank's slab
    m_local = st.size
    torch.cuda.synchronize()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
            torch.cuda.synchronize()

    iters = []
    for _ in range(args.warmup):
        tr = st.step_device(u)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = mp.kernel_launches()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        tr = st.step_device(u)
        iters.append(tr["iterations"])
    ev1.record(stream)
    ev1.synchronize()
    barrier()
    launches = mp.kernel_launches() - launches0
    clk = clocks.stop()
    ms_total = ev0.elapsed_time(ev1)
    t_local = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(t_local, op=torch.distributed.ReduceOp.MAX)
    ms_total = t_local.item()
    ms_step = ms_total / args.steps
    value = m * args.steps / (ms_total * 1e-3)

    # ---- e2e: the public C-ABI call with a HOST (pinned) state buffer, H2D +
    # D2H inside the timed region every step
    u_host = torch.from_numpy(st.initial_state()).pin_memory()
    u_np = u_host.numpy()
    for _ in range(max(1, min(args.warmup, 2))):
        st.step(u_np)
    barrier()
    t0 = time.perf_counter()
    e2e_steps = max(1, min(args.steps, 10))
    for _ in range(e2e_steps):
        st.step(u_np)
    t_e2e = time.perf_counter() - t0
    te = torch.tensor([t_e2e], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
    e2e_value = m * e2e_steps / te.item()

    line = None
    if rank == 0:
        # ---- roofline of the dominant kernel: the FastDiag contraction on the
        # tensor cores (folded 3xTF32, tensor_tc.cu).  Algorithmic work per
        # launch = the reference's contraction: 2 n^4 flop (n^3 outputs x n
        # MACs) and 8 N bytes (x in, out; the diagonal adds 4 N on 1 of 6).
        # Executed: the sine fold halves the MACs and 3xTF32 triples them ->
        # 3 n^4 TF32 flop.  Floors: HBM 8N / peak vs TF32 3n^4 / (bf16 dense / 2);
        # the larger one is the bound reported.
        ms_launch = measure_contraction(mp, torch, st.stream)  # (on a 256^3 grid)
        peaks = load_peaks()
        nk, mk = N_GRID, N_GRID ** 3
        flops = 2.0 * nk ** 4
        bytes_launch = (8.0 * mk * 6 + 4.0 * mk) / 6.0
        tf32 = peaks["bf16_tflops"] / 2.0
        t_hbm = bytes_launch / (peaks["hbm_gbs"] * 1e9)
        t_tc = 3.0 * nk ** 4 / (tf32 * 1e12)
        hbm_gbs_c = bytes_launch / (ms_launch * 1e-3) / 1e9
        tc_exec = 3.0 * nk ** 4 / (ms_launch * 1e-3) / 1e12
        # ---- HBM-bound companion: the step's most frequent stencil, the fused
        # fp32 residual r = b - A x with ||r||^2 (TMA plane pipeline), 12 N bytes
        ktab = kernel_table(mp, N_GRID, peaks["hbm_gbs"])
        sten = ktab["residual_f32"]
        line = {
            "metric": METRIC, "value": value, "unit": "DOF-updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "steps_per_s": 1e3 / ms_step,
            "higher_is_better": True, "scaling": "strong" if split else "weak", "vs_baseline": None,
            "dtype": "f32/f64",
            "data": "synthetic (make_problem: u0 = 0, g = sin sin sin)",
            "config": workload_config(world, split),
            "iterations_per_solve": sorted(set(i for it in iters for i in it)),
            "gpu_launches": launches,
            "e2e": {"value": e2e_value, "unit": "DOF-updates/s", "h2d_bytes_per_step": 8 * m_local * world,
                    "d2h_bytes_per_step": 8 * m_local * world, "steps": e2e_steps,
                    "note": "Stepper.step(host pinned f64 state) through the C-ABI, wall clock"},
            "roofline": {"kernel": "k_tensor_tcf (FastDiag contraction, folded 3xTF32 tcgen05, fp32 accumulate "
                                   "in TMEM)",
                         "bound": "hbm" if t_hbm >= t_tc else "tensor",
                         "achieved": hbm_gbs_c if t_hbm >= t_tc else tc_exec,
                         "peak": peaks["hbm_gbs"] if t_hbm >= t_tc else tf32,
                         "unit": "GB/s" if t_hbm >= t_tc else "TFLOP/s",
                         "frac": hbm_gbs_c / peaks["hbm_gbs"] if t_hbm >= t_tc else tc_exec / tf32,
                         "peak_source": peaks["src"] if t_hbm >= t_tc else peaks["src_tc"] + " / 2 (TF32)",
                         "bytes_per_launch": bytes_launch, "flop_per_launch_algorithmic": flops,
                         "ms_per_launch": ms_launch,
                         "floors_us": {"hbm": t_hbm * 1e6, "tf32_executed": t_tc * 1e6},
                         "tensor_view": {"executed_tf32_tflops": tc_exec, "tf32_dense_peak": tf32,
                                         "frac": tc_exec / tf32,
                                         "algorithmic_fp32_tflops": flops / (ms_launch * 1e-3) / 1e12},
                         "traffic": load_traffic(),
                         "traffic_note": "ncu --set full dram read+write of one launch (profiles/ncu_summary.json)"},
            "roofline_hbm": {"kernel": "k_stencil_tma<LdPlain<float>, EpiResidual> (fp32 7-point residual + norm)",
                             "bound": "hbm", "achieved": sten["gbs"], "peak": peaks["hbm_gbs"], "unit": "GB/s",
                             "frac": sten["frac"], "peak_source": peaks["src"], "bytes_per_launch": sten["bytes"],
                             "ms_per_launch": sten["us"] * 1e-3},
            "clocks": clk,
            "kernels": ktab,
            "kernels_note": (f"each kernel alone on {N_GRID}^3 vectors, CUDA events, algorithmic bytes "
                             "(SURVEY.md §8d) / time vs MEASURED_PEAKS hbm_gbs"),
        }
        if world == 1 and not split and not args.no_variants:
            line["config1_variants"] = config1_variants(mp, torch)
        if not args.no_cpu_baseline and world == 1 and not split:
            budget = float(os.environ.get("MPRKB_CPU_BASELINE_S", "30"))
            threads = os.cpu_count() or 1
            times = reference_steps(N_GRID, 1, budget, threads)
            if times:
                per = sum(times) / len(times)
                line["cpu_baseline"] = {"value": N_GRID ** 3 / per, "unit": "DOF-updates/s", "cores": threads,
                                        "kind": "reference",
                                        "sample": f"{len(times)} step(s) of the same workload, {threads} threads"}
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    if line is not None:
        emit(line)
    return 0


def config1_variants(mp, torch, steps=3):
    """configs[1] reads "fp32-stored CG + block-Jacobi on 1 x B200 vs fp64
    baseline stepper".  The headline runs the reference's own preconditioner
    (FastDiag, the only one its CPU arm has); beside it, the same 256^3 4s3pB
    step with the block-Jacobi extension (b = 8, fp16 block storage, fp32 CG)
    and with the fp64 policy (the "baseline stepper"), device-resident,
    CUDA events on the stepper's stream after one warm-up step."""
    out = {}
    tab = mp.builtin(METHOD)
    for key, kw, note in (
            ("cg_block_jacobi_b8_f16", dict(prec="f32", tol=TOL, max_iter=400, preconditioner="block-jacobi",
                                            block_size=8, block_storage="f16"),
             "fp32 stages, CG + block-Jacobi (x-line blocks of 8, fp16 storage), pipelined FAST CG"),
            ("fp64_baseline_stepper", dict(prec="f64", tol=1e-5, max_iter=MAX_ITER),
             "fp64 stages, CG + FastDiag on CUDA cores (the fp64 policy)")):
        prec, tol, mi = kw.pop("prec"), kw.pop("tol"), kw.pop("max_iter")
        st = mp.Stepper("heat", N_GRID, tab, TAU, tol, prec, mi, **kw)
        s = torch.cuda.ExternalStream(st.stream)
        u = torch.from_numpy(st.initial_state()).cuda()
        st.step_device(u)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        its = []
        a.record(s)
        for _ in range(steps):
            its.append(st.step_device(u)["iterations"])
        b.record(s)
        b.synchronize()
        ms = a.elapsed_time(b) / steps
        out[key] = {"ms_per_step": ms, "value": N_GRID ** 3 / (ms * 1e-3), "unit": "DOF-updates/s",
                    "iterations_per_solve": its, "tol": tol, "steps": steps, "note": note}
        del st
    out["fp64_baseline_stepper"]["contraction"] = fp64_contraction_roofline(mp)
    return out


def fp64_contraction_roofline(mp, reps=10):
    """The fp64 stepper's dominant kernel, the sine-folded FastDiag
    contraction on the FP64 tensor cores (k_tensor_dmma, mma.sync m16n8k8
    .f64), timed alone per side at 256^3 against the measured DMMA peak
    (csrc/peak.cu): n N / 2 executed FMAs = n N flop per launch (the fold
    halves the 2 n N algorithmic flop).  The CUDA-core DFMA peak is
    reported beside it (the DFMA kernel it replaced: profiles/r02)."""
    import ctypes as C

    peak = mp_fma_peak(mp, 2)
    dfma_peak = mp_fma_peak(mp, 1)
    n = N_GRID
    flop = float(n) * n ** 3  # folded: n/2 rows x n q per output pair = n N / 2 FMAs = n N flop
    sides = {}
    for sd in "RML":
        ms, by = C.c_double(), C.c_double()
        mp.check(mp._c.lib.mprkb_kernel_bench(f"tensor_f64_{sd}".encode(), n, reps, C.byref(ms), C.byref(by)))
        tf = flop / (ms.value * 1e-3) / 1e12
        sides[sd] = {"us": round(ms.value * 1e3, 2), "executed_tflops": round(tf, 2), "frac": round(tf / peak, 3)}
    return {"kernel": "k_tensor_dmma (sine-folded fp64 GEMM on the FP64 tensor cores, mma.sync m16n8k8)",
            "bound": "fp64 tensor (DMMA)", "peak_tflops": round(peak, 2),
            "peak_source": "csrc/peak.cu independent DMMA chains, one wave, measured here",
            "dfma_peak_tflops": round(dfma_peak, 2), "executed_flop_per_launch": flop, "sides": sides}


KERNELS = ["copy_f32", "stencil_f64", "stencil_f32", "residual_f32", "apply_dot_f32", "dots2_f32", "cg_fused_f32",
           "cg_fused_self_f32",
           "apply_f64", "apply_f32", "dot_f32", "cg_update_f32", "combine_7", "final_4", "block_jacobi_f16", "cg_bj_f16",
           "csr_f32", "csr_f16"]


def kernel_table(mp, n, peak_gbs, reps=20):
    """HBM-bound kernels of the step (and the SpMV / block-Jacobi extensions)
    timed alone on n^3 vectors: achieved algorithmic GB/s and fraction of the
    measured copy peak — the 'SpMV HBM GB/s' half of BASELINE.json's metric."""
    import ctypes as C

    out = {}
    for k in KERNELS:
        ms, by = C.c_double(), C.c_double()
        mp.check(mp._c.lib.mprkb_kernel_bench(k.encode(), n, reps, C.byref(ms), C.byref(by)))
        gbs = by.value / (ms.value * 1e-3) / 1e9
        out[k] = {"us": round(ms.value * 1e3, 2), "bytes": by.value, "gbs": round(gbs, 1),
                  "frac": round(gbs / peak_gbs, 4)}
    return out


def mp_fma_peak(mp, dtype):
    import ctypes as C

    v = C.c_double()
    mp.check(mp._c.lib.mprkb_measure_fma_peak(dtype, C.byref(v)))
    return v.value


def measure_stencil(mp, torch, stream_ptr, reps=20):
    n = N_GRID
    x = torch.randn(n ** 3, dtype=torch.float64, device="cuda")
    A = mp.Operator.stencil(1, n, 0, 1.0, -1.0)
    s = torch.cuda.ExternalStream(stream_ptr)
    with torch.cuda.stream(s):
        for _ in range(3):
            A.apply(x)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            A.apply(x)
        b.record(s)
        b.synchronize()
    return a.elapsed_time(b) / reps


def load_peaks():
    out = {"hbm_gbs": 6650.0, "src": "B200_PROFILING.md fallback", "bf16_tflops": 2250.0,
           "src_tc": "nominal bf16 dense (no MEASURED_PEAKS.json)"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        out.update(hbm_gbs=float(d["hbm_gbs"]), src="MEASURED_PEAKS.json hbm_gbs (measured copy)")
        out.update(bf16_tflops=float(d["bf16_tflops"]), src_tc="MEASURED_PEAKS.json bf16_tflops (burst)")
    except (OSError, ValueError, KeyError):
        pass
    return out


# The driver parses ONE JSON line from stdout.  Libraries print to the C-level
# stdout on their own (NCCL's "NCCL version ..." banner at communicator init,
# whatever a dlopen'ed library printf's), so the process's fd 1 is pointed at
# stderr for the whole run and only emit() writes to the original stdout.
_STDOUT_FD = None


def _isolate_stdout():
    global _STDOUT_FD
    if _STDOUT_FD is None:
        sys.stdout.flush()
        _STDOUT_FD = os.dup(1)
        os.dup2(2, 1)


def emit(obj):
    data = (json.dumps(obj) + "\n").encode()
    if _STDOUT_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_STDOUT_FD, data)


def main():
    _isolate_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--no-variants", action="store_true", help="skip the configs[1] companion steppers")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--split", action="store_true",
                    help="configs[2] path (512^3 through the NCCL split stepper) even on one GPU")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_cuda_arm(args)


if __name__ == "__main__":
    sys.exit(main())
