#!/usr/bin/env python
"""bench.py -- BASELINE.json metric: fused kernel-pair executions/s (fp64)
and HBM GB/s vs the roofline, with the reference CPU executor beside it.

Workload (config.workload): BASELINE config 5, the largest single-GPU
configuration -- forward L z = b then backward L^T x = z on the 27-point
128^3 stencil (n = 2,097,152, nnz(L) = 28,920,060), BASELINE's batch of 8
systems (own diagonal perturbation and right-hand side each), one fused
launch per step.  One "exec" = one fused kernel-pair execution on one system.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

With --gpus N > 1 and no torchrun environment, bench.py launches its N ranks
itself (torch.distributed.run, 127.0.0.1); under torchrun WORLD_SIZE must
equal N.  Multi-GPU: the batch of 8 is sharded, 8/N systems per GPU
(strong scaling; the systems are independent, so there is no data-path
collective -- torch.distributed only provides the barrier and the
max-over-ranks of the timings); ``--systems-per-gpu K`` runs K systems on
every GPU instead (weak scaling), and at N > 1 the line also carries that
weak-scaling measurement with K = 8.  ``--config 1 --shard-spmv`` runs
config 1 with the solve on rank 0 and the SpMV rows sharded over the ranks
(one point-to-point x exchange + a y all-gather over NCCL; strong scaling).

The reference arm (--impl reference) runs only oracle/_ref (the unmodified
reference compiled from /root/reference, plus the repo's input generators
compiled into it) and never imports this package or loads libsfgpu.so.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused kernel-pair execs/s (fp64)"
UNIT = "execs/s"
CONFIG_COMBO = {1: 4, 2: 5, 3: 6, 4: 7, 5: 8}
CONFIG_NAME = {
    1: "SpTRSV->SpMV 2-D 5-pt 512^2 (combo 4)",
    2: "SpIC0->SpTRSV 3-D 7-pt 64^3 (combo 5)",
    3: "SpILU0->SpTRSV 3-D conv-diff 96^3 (combo 6)",
    4: "DAD->SpIC0 random band n=1e6 (combo 7)",
    5: "SpTRSV->SpTRSV^T fwd L, bwd L^T, 27-pt 128^3, batch of 8 systems",
}


# ---------------------------------------------------------------------------
# plumbing: ranks, barrier, max over ranks, clocks
# ---------------------------------------------------------------------------
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch
            import torch.distributed as td
            backend = "nccl" if torch.cuda.is_available() else "gloo"
            if backend == "nccl":
                torch.cuda.set_device(self.local)
            td.init_process_group(backend=backend)
            self.td = td
            self.torch = torch
            self.dev = torch.device("cuda", self.local) if backend == "nccl" else torch.device("cpu")

    def barrier(self):
        if self.world > 1:
            self.td.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.td.destroy_process_group()


REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
           0x2: "applications_clocks_setting", 0x10: "sync_boost"}


class ClockSampler:
    """NVML sampling of the SM clock and throttle reasons while running."""

    def __init__(self, index: int, period_s: float = 0.005):
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self.ok = False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self.period = period_s

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(v for k, v in REASONS.items() if self.reasons & k),
                "samples": len(self.samples)}


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(workload: str):
    """dram bytes per launch of the dominant kernel from the committed ncu
    capture (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(workload)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# algorithmic bytes (each array once per direction)
# ---------------------------------------------------------------------------
def algorithmic_bytes(cfg: int, n: int, nnzL: int, nnzA: int) -> int:
    ptr = 4 * (n + 1)
    vec = 8 * n
    if cfg == 1:  # read L + read A + read b + write x + write y
        return (ptr + 12 * nnzL) + (ptr + 12 * nnzA) + 3 * vec
    if cfg == 2:  # read A_lower + write L.val + read b + write z
        return ptr + 12 * nnzL + 8 * nnzL + 2 * vec
    if cfg == 3:  # read A + write LU.val + read b + write z
        return ptr + 12 * nnzA + 8 * nnzA + 2 * vec
    if cfg == 4:  # read A_lower + write L.val + write d
        return ptr + 12 * nnzL + 8 * nnzL + vec
    if cfg == 5:  # per system: read L once + read b + write z + write x
        return ptr + 12 * nnzL + 3 * vec
    raise ValueError(cfg)


def physical_bytes(cfg: int, n: int, nnzL: int, nnzA: int, S: int) -> int:
    """Bytes the executor must move at least (config 5: each system's L values
    streamed by both solves, the shared pattern twice, b read, z written and
    re-read, x written); the other configs equal the algorithmic bytes."""
    if cfg != 5:
        return algorithmic_bytes(cfg, n, nnzL, nnzA)
    ptr = 4 * (n + 1)
    return S * (2 * 8 * nnzL + 4 * 8 * n) + 2 * (4 * nnzL + ptr)


def unique_bytes(cfg: int, n: int, nnzL: int, nnzA: int, S: int) -> int:
    """Algorithmic bytes of one launch with the pattern shared by the S
    systems counted once (config 5: row pointers and column indices once,
    values and vectors per system)."""
    if cfg != 5:
        return algorithmic_bytes(cfg, n, nnzL, nnzA)
    return 4 * (n + 1) + 4 * nnzL + S * (8 * nnzL + 3 * 8 * n)


def kernel_name(cfg: int, combo: int, S: int) -> str:
    G = 4 if S <= 8 else 32 // S  # chain_G (csrc/chain.cuh)
    if cfg == 5 and S == 1:  # 27-point rows: one warp per chain (plan.cu executor choice)
        return f"k_chain<1,{G},12,{combo}> (fwd L + bwd L^T)"
    if S == 1 and combo in (1, 2, 4, 8):  # single systems: multi-line step-stream executor
        return {4: "k_mline1 (fwd L + SpMV row blocks)", 2: "k_mline1 (SpMV blocks + fwd L)"}.get(
            combo, f"k_mline1 (combo {combo})")
    return {8: f"k_chain_sm<{S},{G},12,8> (fwd L + bwd L^T)", 1: f"k_chain_sm<{S},{G},12,1> (fwd L + fwd L)",
            5: "k_ic0_pipe (task records, operands one task ahead)", 6: "k_ilu0_pack<6,4,8> (4 rows per warp)",
            3: "k_ilu0_pack<3,4,8> (4 rows per warp)",
            7: "k_ic0_warp<7>"}.get(combo, f"combo {combo} executor")


def copy_bound(h2d_bytes: int, d2h_bytes: int, device: int, reps: int = 5):
    """The PCIe floor of one e2e step: the step's input copy and its output
    copy issued together on two streams from/to page-locked memory (the
    best the overlapped e2e pipeline can do), median of reps."""
    try:
        import torch
        dev = torch.device("cuda", device)
        hi = torch.empty(max(h2d_bytes, 8) // 8, dtype=torch.float64, pin_memory=True)
        ho = torch.empty(max(d2h_bytes, 8) // 8, dtype=torch.float64, pin_memory=True)
        di = torch.empty(hi.numel(), dtype=torch.float64, device=dev)
        do = torch.zeros(ho.numel(), dtype=torch.float64, device=dev)
        s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

        def timed(h2d, d2h):
            t = []
            for _ in range(reps):
                torch.cuda.synchronize(dev)
                t0 = time.perf_counter()
                if h2d:
                    with torch.cuda.stream(s1):
                        di.copy_(hi, non_blocking=True)
                if d2h:
                    with torch.cuda.stream(s2):
                        ho.copy_(do, non_blocking=True)
                torch.cuda.synchronize(dev)
                t.append(time.perf_counter() - t0)
            return statistics.median(t)
        th, td, tb = timed(True, False), timed(False, True), timed(True, True)
        return {"h2d_gbs": h2d_bytes / th / 1e9, "d2h_gbs": d2h_bytes / td / 1e9,
                "both_ms": tb * 1e3, "method": "torch copies from/to pinned memory, "
                "the step's input and output issued together on two streams"}
    except Exception as e:  # a missing torch/CUDA only drops the annotation
        return {"error": str(e)[:200]}


def workload_config(cfg: int, combo: int, n: int, nnzA: int, nnzL: int, S: int, world: int):
    """The `config` object of a bench line: the same dict for our arm and for
    the reference arm, so the driver can match them key by key."""
    name = CONFIG_NAME[cfg]
    if cfg == 5 and combo == 1:
        name = name.replace("bwd L^T", "fwd L (combo 1 parity mode)")
    return {"workload": name, "baseline_config": cfg, "combo": combo, "n": n, "nnz_A": nnzA,
            "nnz_L": nnzL, "systems_per_gpu": S, "global_systems": S * world,
            "l2": ("inputs larger than L2 (L values+indices %.2f GB/GPU > 126 MB)"
                   % (S * 12 * nnzL / 1e9)) if cfg == 5 else "see DESIGN.md",
            "parallelism": f"dp{world} (independent systems, no collective)"}


def lower_nnz(M) -> int:
    cols = np.repeat(np.arange(M.n, dtype=np.int64), np.diff(M.colptr))
    return int(np.count_nonzero(M.rowidx >= cols))


# ---------------------------------------------------------------------------
# inputs
# ---------------------------------------------------------------------------
def make_inputs(cfg: int, size, nsys: int, sys0: int):
    import paper_2111_12238_b200 as sf
    if cfg == 5:
        M, vals = sf.config5_systems(size=size, nsys=nsys, seed0=1000 + sys0)
        vin = np.concatenate([sf.gen_vector(M.n, 7 + sys0 + s) for s in range(nsys)])
        return M, vals, vin
    M = sf.config_matrix(cfg, size=size)
    vin = sf.gen_vector(M.n, 7)
    return M, None, vin


# ---------------------------------------------------------------------------
# the reference CPU executor (oracle/_ref: unmodified reference headers).
# Inputs come from oracle/_ref too (the repo's generators compiled into it),
# so these legs never load libsfgpu.so.
# ---------------------------------------------------------------------------
def ref_inputs(ref, cfg: int, size, nsys: int = 1, sys0: int = 0):
    if cfg == 5:
        M, vals = ref.config_matrix(5, size, nsys_perturb=nsys, seed0=1000 + sys0)
        vin = np.concatenate([ref.gen_vector(M.n, 7 + sys0 + s) for s in range(nsys)])
        return M, vals, vin
    M = ref.config_matrix(cfg, size)
    return M, None, ref.gen_vector(M.n, 7)


def reference_fused(cfg: int, M, vin, nthreads: int, warmups: int, repeats: int):
    """Times the reference's execute_fused (msp + compile_schedule once, then
    warmups + repeats) for configs 1-4 (the reference's own combos)."""
    from oracle.oracle import Csc, Reference
    ref = Reference()
    combo = CONFIG_COMBO[cfg]
    st = ref.state(combo, Csc(M.n, M.colptr, M.rowidx, M.values), 7, vin=vin[:M.n])
    t0 = time.perf_counter()
    times, insp, nsp = st.bench(1, nthreads, warmups, repeats)
    wall = time.perf_counter() - t0
    return {"times": times.tolist(), "median_s": float(np.median(times)), "inspector_s": insp,
            "s_partitions": nsp, "combo": combo, "wall_s": wall}


class RefConfig5:
    """Config 5 (fwd L z = b, then bwd L^T x = z) on the reference's own
    parallel executor.  The reference has no backward solve and no such
    pair, so each system's two solves run as single kernels -- kernel 1 of a
    combo-1 KernelState under its LBC schedule, executed by execute_unfused
    (executor.hpp:325-381) with an empty kernel-2 schedule -- the backward
    one on permute_symmetric(transpose(L), rev) (matrix.hpp:130-173) with z
    reversed, exactly SURVEY.md 8(c)'s composition.  The systems share the
    pattern, so the DAG and LBC schedule are built once per direction and
    each system's state differs only on its diagonal.  A step's time is the
    sum of the executor wall times (ExecStats::wall_ns) of its solves."""

    def __init__(self, ref, M, vals, vin, nsys: int, nthreads: int):
        from oracle.oracle import Csc
        self.n, self.nsys, self.vin = M.n, nsys, vin
        n = M.n
        cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(M.colptr))
        dpos = np.nonzero(M.rowidx == cols)[0]
        t0 = time.perf_counter()
        M0 = Csc(n, M.colptr, M.rowidx, vals[:M.nnz])
        f0 = ref.solver(M0, nthreads)
        b0 = ref.solver(ref.backward_matrix(M0), nthreads)
        self.inspector_s = f0.inspector_s + b0.inspector_s
        self.fwd, self.bwd = [f0], [b0]
        for s in range(1, nsys):
            d = vals[s * M.nnz:(s + 1) * M.nnz][dpos]
            self.fwd.append(f0.with_diagonal(d))
            self.bwd.append(b0.with_diagonal(d[::-1].copy()))
        self.setup_s = time.perf_counter() - t0
        self.z = np.empty(n)
        self.xr = np.empty(n)

    def step(self, out=None) -> float:
        n, secs = self.n, 0.0
        for s in range(self.nsys):
            secs += self.fwd[s].run(self.vin[s * n:(s + 1) * n], self.z)
            secs += self.bwd[s].run(self.z[::-1].copy(), self.xr)
            if out is not None:
                out[s, :n] = self.z
                out[s, n:] = self.xr[::-1]
        return secs


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
GLOBAL_BATCH = 8  # BASELINE.json configs[4]: a batch of 8 independent systems


def systems_per_gpu(args, D) -> int:
    """Config 5: BASELINE's batch of 8 sharded over the ranks (8/N each), or
    --systems-per-gpu K on every rank (weak scaling)."""
    if args.systems_per_gpu is not None:
        return args.systems_per_gpu
    if GLOBAL_BATCH % D.world:
        raise SystemExit(f"the batch of {GLOBAL_BATCH} does not split over {D.world} GPUs; "
                         "pass --systems-per-gpu")
    return GLOBAL_BATCH // D.world


def scaling_kind(args, cfg, D) -> str:
    return "weak" if (cfg == 5 and args.systems_per_gpu is not None) else "strong"


def check_result(st, cfg, combo, M, vals, vin, S):
    """Bit-exact check of the plan's last execution (system 0) against the
    oracle -- the result the timed loop produced."""
    from oracle.oracle import Csc, Oracle
    orc = Oracle()
    n = M.n
    v0 = M.values if vals is None else vals[:M.nnz]
    want = orc.run_sequential(combo, Csc(n, M.colptr, M.rowidx, v0), 7, vin=vin[:n])
    got = st.collect_outputs()[:len(want)]
    return {"checked": "system 0 of this rank's batch vs oracle/sf_oracle.c",
            "bit_exact": bool(np.array_equal(got, want))}


def run_ours(args, D: Dist):
    import paper_2111_12238_b200 as sf
    from paper_2111_12238_b200 import abi
    abi.set_device(D.local)
    cfg = args.config
    combo = CONFIG_COMBO[cfg] if not (cfg == 5 and args.mode == "fwdfwd") else 1
    S = systems_per_gpu(args, D) if cfg == 5 else 1
    t0 = time.perf_counter()
    M, vals, vin = make_inputs(cfg, args.size, S, D.rank * S)
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    st = sf.make_state(combo, M, seed=7, nsys=S, values=vals, vin=vin)
    t_state = time.perf_counter() - t0
    t0 = time.perf_counter()
    st.inspect()
    t_insp = time.perf_counter() - t0
    nnzL = lower_nnz(M)
    bytes_per_launch = algorithmic_bytes(cfg, M.n, nnzL, M.nnz) * S

    # ---- device-resident throughput (value)
    if args.warmup > 0:
        st.bench(args.warmup)
    D.barrier()
    launches0 = st.launch_count()
    with ClockSampler(D.local) as clk:
        total_ms, kernel_ms = st.bench(args.steps)
    launches = st.launch_count() - launches0
    D.barrier()
    ms_step = D.max(total_ms / args.steps)
    kernel_ms = D.max(kernel_ms)
    value = S * D.world / (ms_step / 1e3)

    # ---- unfused two-kernel GPU sequence on the same inputs
    st.bench(max(1, args.warmup), unfused=True)
    D.barrier()
    u_total, u_kernel = st.bench(args.steps, unfused=True)
    D.barrier()
    u_ms = D.max(u_total / args.steps)

    # ---- the joint-DAG wavefront executor (execute_joint_wavefront, the
    # paper's level-set baseline) on the same inputs
    st.bench(max(1, args.warmup), unfused=2)
    D.barrier()
    w_total, w_kernel = st.bench(args.steps, unfused=2)
    D.barrier()
    w_ms = D.max(w_total / args.steps)
    w_levels = int(st.wavefront().nlevels())

    # ---- end to end through the public API: H2D of the step's inputs, the
    # execution, D2H of the step's outputs.  Solve pairs go through
    # sfg_execute_batch, which overlaps step k+1's input copy and step k-1's
    # output copy with step k; factorization pairs re-upload the matrix
    # values (their input) and b with set_values / set_vin each step.
    n = M.n
    factor = combo in (5, 6, 7)
    has_vin = combo != 7
    pin_val = abi.PinnedArray(S * M.nnz) if factor else None
    if factor:
        pin_val.array[:] = M.values if vals is None else vals
    NB = 3  # distinct page-locked buffers, reused round robin
    pins_in = [abi.PinnedArray(S * n) for _ in range(NB)] if has_vin else []
    # solve pairs return kernel 2's output (the solution) per step; the
    # factorization pairs return the collect_outputs layout
    out_len = n if not factor else st.output_len
    pins_out = [abi.PinnedArray(S * out_len) for _ in range(NB)]
    for pa in pins_in:
        pa.array[:] = vin

    if factor:
        def e2e_run(k):
            for i in range(k):
                st.set_values(pin_val.array)
                if has_vin:
                    st.set_vin(pins_in[i % NB].array)
                st.execute_fused(sync=False)
                st.collect_outputs(pins_out[i % NB].array)
        path = ("sfg_set_values + " + ("sfg_set_vin + " if has_vin else "")
                + "sfg_execute_fused + sfg_collect_outputs per step, pinned host buffers")
    else:
        def e2e_run(k):
            st.execute_batch([pins_in[i % NB].array for i in range(k)],
                             [pins_out[i % NB].array for i in range(k)], final_only=True)
        path = ("sfg_execute_batch_ex(SFG_OUTPUTS_FINAL): each step copies its right-hand "
                "sides in and its solutions (kernel 2's output) out, H2D of step k+1 and D2H "
                "of step k-1 overlapped with step k; pinned host buffers")

    e2e_run(max(1, args.warmup))
    D.barrier()
    with ClockSampler(D.local) as clk_e2e:
        t0 = time.perf_counter()
        e2e_run(args.steps)
        e2e_s = (time.perf_counter() - t0) / args.steps
    D.barrier()
    e2e_s = D.max(e2e_s)
    h2d = 8 * S * ((n if has_vin else 0) + (M.nnz if factor else 0))
    e2e = {"value": S * D.world / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": 8 * S * out_len, "ms_per_step": e2e_s * 1e3,
           "path": path}
    # the step's own copies are its floor (they overlap the kernel)
    cb = copy_bound(h2d, 8 * S * out_len, D.local)
    if "both_ms" in cb:
        cb["frac_of_step"] = cb["both_ms"] / (e2e_s * 1e3)
    e2e["copy_floor"] = cb

    # ---- the timed execution's result against the oracle (system 0 of the
    # rank; the plan's outputs are those of its last execution)
    parity = check_result(st, cfg, combo, M, vals, vin, S)
    peak, peak_src = hbm_peak()
    achieved = bytes_per_launch / (kernel_ms / 1e3) / 1e9
    workload = f"config{cfg}"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": D.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": scaling_kind(args, cfg, D), "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(cfg, combo, M.n, M.nnz, nnzL, S, D.world),
        "parity": parity,
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(workload),
                     "peak_source": peak_src, "kernel_ms": kernel_ms,
                     "algorithmic_bytes_per_launch": bytes_per_launch,
                     "kernel": kernel_name(cfg, combo, S),
                     "physical_bytes_per_launch": physical_bytes(cfg, M.n, nnzL, M.nnz, S),
                     "physical_frac": physical_bytes(cfg, M.n, nnzL, M.nnz, S)
                     / (kernel_ms / 1e3) / 1e9 / peak,
                     # the shared pattern counted once instead of once per system
                     "unique_bytes_per_launch": unique_bytes(cfg, M.n, nnzL, M.nnz, S),
                     "unique_frac": unique_bytes(cfg, M.n, nnzL, M.nnz, S)
                     / (kernel_ms / 1e3) / 1e9 / peak},
        "unfused": {"ms_per_step": u_ms, "value": S * D.world / (u_ms / 1e3),
                    "fused_speedup": u_ms / ms_step},
        "wavefront": {"ms_per_step": w_ms, "value": S * D.world / (w_ms / 1e3),
                      "levels": w_levels, "fused_speedup": w_ms / ms_step,
                      "executor": "joint-DAG level sets, grid barrier per level (sfg_execute_wavefront)"},
        "e2e": e2e,
        "clocks": clk.summary(),
        "clocks_e2e": clk_e2e.summary(),
        "setup_s": {"generate": t_gen, "make_state": t_state, "inspect_gpu": t_insp},
    }

    # ---- CPU baseline: the reference's fused executor on the box's host cores
    if D.world == 1 and D.rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, args.size)

    # ---- weak scaling beside the sharded batch: 8 systems on every GPU
    if D.world > 1 and cfg == 5 and args.systems_per_gpu is None and not args.no_extras:
        Mw, valsw, vinw = make_inputs(5, args.size, GLOBAL_BATCH, D.rank * GLOBAL_BATCH)
        sw = sf.make_state(8, Mw, seed=7, nsys=GLOBAL_BATCH, values=valsw, vin=vinw).inspect()
        sw.bench(args.warmup)
        D.barrier()
        wt, _ = sw.bench(args.steps)
        D.barrier()
        wms = D.max(wt / args.steps)
        line["weak_scaling"] = {"systems_per_gpu": GLOBAL_BATCH, "global_systems": GLOBAL_BATCH * D.world,
                                "ms_per_step": wms, "value": GLOBAL_BATCH * D.world / (wms / 1e3),
                                "scaling": "weak"}
        sw.close()

    # ---- the other BASELINE configs on this GPU (single GPU only)
    if D.world == 1 and not args.no_extras and cfg == 5:
        line["other_configs"] = other_configs(args)

    for pa in [pin_val] + pins_in + pins_out:
        if pa is not None:
            pa.free()
    st.close()
    return line


# ---------------------------------------------------------------------------
# config 1 split across ranks: rank 0 solves, x slices travel
# point-to-point over NCCL, every rank computes its rows of y, all-gather
# ---------------------------------------------------------------------------
def run_sharded(args, D: Dist):
    import torch
    import paper_2111_12238_b200 as sf
    from paper_2111_12238_b200 import abi, shard
    abi.set_device(D.local)
    torch.cuda.set_device(D.local)
    M = sf.config_matrix(1, size=args.size)
    n = M.n
    vin = sf.gen_vector(n, 7)
    st = sf.make_state(4, M, seed=7, vin=vin)
    st.inspect()
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        st.set_stream(stream.cuda_stream)
        solve, spmv = shard.plan_callbacks(st, n)
        if D.rank != 0:
            solve = None
        rowptr, colidx = shard.csr_pattern(M.colptr, M.rowidx, n)
        S = shard.ShardedSpmv(getattr(D, "td", None), D.rank, D.world, n, rowptr, colidx,
                              torch.device("cuda", D.local), solve=solve, spmv=spmv)
        for _ in range(args.warmup):
            S.step()
        stream.synchronize()
        D.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = st.launch_count()
        with ClockSampler(D.local) as clk:
            e0.record(stream)
            for _ in range(args.steps):
                y = S.step()
            e1.record(stream)
            e1.synchronize()
        launches = st.launch_count() - l0
        D.barrier()
        ms = D.max(e0.elapsed_time(e1) / args.steps)
        y_dev = y.cpu().numpy()

        # e2e: b from pinned host memory into the plan (rank 0), y back to host
        pin_b = abi.PinnedArray(n)
        pin_b.array[:] = vin
        y_host = torch.empty(n, dtype=torch.float64, pin_memory=True)
        D.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            if D.rank == 0:
                st.set_vin(pin_b.array)
            y_host.copy_(S.step(), non_blocking=True)
            stream.synchronize()
        e2e_s = D.max((time.perf_counter() - t0) / args.steps)
        pin_b.free()
    st.set_stream(None)
    # parity of the timed result: the single-GPU fused combo 4 on rank 0
    parity = None
    if D.rank == 0:
        ref = sf.make_state(4, M, seed=7, vin=vin)
        ref.execute_fused()
        want = ref.collect_outputs()[n:2 * n]
        parity = bool(np.array_equal(y_dev, want) and np.array_equal(y_host.numpy(), want))
        ref.close()
    nnzL = lower_nnz(M)
    peak, peak_src = hbm_peak()
    abytes = algorithmic_bytes(1, n, nnzL, M.nnz)
    st.close()
    return {
        "metric": METRIC, "value": 1e3 / ms, "unit": UNIT, "n_gpus": D.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": CONFIG_NAME[1] + ", SpMV rows sharded over ranks",
                   "baseline_config": 1, "combo": 4, "n": n, "nnz_A": M.nnz,
                   "shards": S.shards, "x_ranges": S.ranges,
                   "halo_rows": shard.halo_rows(S.shards, S.ranges),
                   "exchange_bytes_per_step": S.exchanged_bytes(),
                   "l2": "not flushed (whole working set %.1f MB < L2)" % (abytes / 1e6),
                   "parallelism": f"solve on rank 0, SpMV row-sharded over {D.world} ranks"},
        "gpu_launches": launches, "parity_vs_fused": parity,
        "roofline": {"bound": "hbm", "achieved": abytes / (ms / 1e3) / 1e9, "peak": peak,
                     "unit": "GB/s", "frac": abytes / (ms / 1e3) / 1e9 / peak, "traffic": None,
                     "peak_source": peak_src, "kernel": "whole step (solve + sharded SpMV)"},
        "e2e": {"value": 1.0 / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n, "ms_per_step": e2e_s * 1e3},
        "clocks": clk.summary(),
    }


def cpu_baseline(cfg, size):
    """The reference on this box's host cores, a bounded sample of the
    workload (inputs generated by oracle/_ref, not by this package)."""
    from oracle.oracle import Reference
    T = cpu_threads()
    if not Reference.available():
        from oracle.oracle import Csc, Oracle
        import paper_2111_12238_b200 as sf
        M = sf.config_matrix(cfg, size=size) if cfg != 5 else sf.config5_systems(size=size, nsys=1)[0]
        orc = Oracle()
        t0 = time.perf_counter()
        orc.run_sequential(CONFIG_COMBO[cfg], Csc(M.n, M.colptr, M.rowidx, M.values), 7)
        dt = time.perf_counter() - t0
        return {"value": 1.0 / dt, "unit": UNIT, "cores": 1, "kind": "port",
                "sample": "1 system, oracle sequential restatement (make_state included)"}
    ref = Reference()
    if cfg == 5:
        M, vals, vin = ref_inputs(ref, 5, size, 1, 0)
        r = RefConfig5(ref, M, vals, vin, 1, T)
        r.step()  # warm-up
        times = [r.step() for _ in range(3)]
        med = float(np.median(times))
        return {"value": 1.0 / med, "unit": UNIT, "cores": T, "kind": "reference",
                "sample": ("1 system of the batch (fwd L then bwd L^T on the reference's "
                           f"parallel executor, T={T}, LBC schedules built once), median of 3 "
                           "after 1 warm-up"),
                "ms_per_exec": med * 1e3, "inspector_s": r.inspector_s}
    M, _, vin = ref_inputs(ref, cfg, size)
    r = reference_fused(cfg, M, vin, T, warmups=1, repeats=3)
    return {"value": 1.0 / r["median_s"], "unit": UNIT, "cores": T, "kind": "reference",
            "sample": (f"reference execute_fused (msp + compile_schedule, T={T}), median of "
                       f"{len(r['times'])} after 1 warm-up"),
            "ms_per_exec": r["median_s"] * 1e3, "inspector_s": r["inspector_s"],
            "s_partitions": r["s_partitions"]}


def other_configs(args):
    import paper_2111_12238_b200 as sf
    from oracle.oracle import Reference
    out = {}
    peak, _ = hbm_peak()
    T = cpu_threads()
    for cfg in (1, 2, 3, 4):
        M, _, vin = make_inputs(cfg, None, 1, 0)
        combo = CONFIG_COMBO[cfg]
        st = sf.make_state(combo, M, seed=7).inspect()
        reps = 20
        st.bench(3)
        tot, ker = st.bench(reps)
        ut, uk = st.bench(reps, unfused=True)
        st.bench(2, unfused=2)
        wt, wk = st.bench(reps, unfused=2)
        nnzL = lower_nnz(M)
        byts = algorithmic_bytes(cfg, M.n, nnzL, M.nnz)
        ms = tot / reps
        rec = {"workload": CONFIG_NAME[cfg], "n": M.n, "nnz": M.nnz,
               "value": 1e3 / ms, "ms_per_exec": ms, "kernel_ms": ker,
               "achieved_gbs": byts / (ker / 1e3) / 1e9,
               "frac": byts / (ker / 1e3) / 1e9 / peak,
               "unfused_ms_per_exec": ut / reps, "fused_speedup": (ut / reps) / ms,
               "wavefront_ms_per_exec": wt / reps, "speedup_vs_wavefront": (wt / reps) / ms,
               # level_info(joint_dag) (dag.hpp:197-218) and the executor's own
               # dependency levels (s-partitions of its FusedPartitioning)
               "critical_path": int(st.level_info(3).critical_path),
               "executor_levels": int(st.partitioning().b()),
               "traffic": ncu_traffic(f"config{cfg}")}
        if Reference.available() and not args.no_cpu_baseline:
            try:
                r = reference_fused(cfg, M, vin, T, warmups=1, repeats=3)
                rec["cpu_reference"] = {"value": 1.0 / r["median_s"], "cores": T,
                                        "ms_per_exec": r["median_s"] * 1e3,
                                        "inspector_s": r["inspector_s"]}
            except Exception as e:  # keep the bench line even if the CPU leg fails
                rec["cpu_reference"] = {"error": str(e)[:200]}
        # NER (bench.hpp:29-36): executions that amortise this GPU's
        # inspection (make_state + inspect) against the CPU reference
        t0 = time.perf_counter()
        st2 = sf.make_state(combo, M, seed=7).inspect()
        insp = time.perf_counter() - t0
        st2.close()
        rec["inspector_s"] = insp
        cpu = rec.get("cpu_reference", {}).get("ms_per_exec")
        if cpu:
            rec["ner_vs_cpu_reference"] = (insp / ((cpu - ms) / 1e3)) if cpu > ms else None
        out[f"config{cfg}"] = rec
        st.close()
    # config 5's systems under the reference's own combo 1 (fwd L -> fwd L, the
    # pair the CPU baseline times): its joint DAG lets the second solve trail
    # the first, so fused should beat the unfused two-launch sequence
    S = args.systems_per_gpu or GLOBAL_BATCH
    M, vals, vin = make_inputs(5, args.size, S, 0)
    st = sf.make_state(1, M, seed=7, nsys=S, values=vals, vin=vin).inspect()
    reps = 20
    st.bench(3)
    tot, ker = st.bench(reps)
    st.bench(3, unfused=True)
    ut, _ = st.bench(reps, unfused=True)
    nnzL = lower_nnz(M)
    byts = algorithmic_bytes(5, M.n, nnzL, M.nnz) * S
    out["config5_fwdfwd"] = {"workload": CONFIG_NAME[5].replace("bwd L^T", "fwd L (combo 1)"),
                             "systems": S, "value": S * reps / (tot / 1e3),
                             "ms_per_exec": tot / reps, "kernel_ms": ker,
                             "achieved_gbs": byts / (ker / 1e3) / 1e9,
                             "frac": byts / (ker / 1e3) / 1e9 / peak,
                             "unfused_ms_per_exec": ut / reps, "fused_speedup": ut / tot}
    st.close()
    # the iterative solver the executors serve: PCG with the IC0
    # factor (combo 5) and the fused forward/backward solve (combo 8) as M^-1
    M = sf.config_matrix(2)
    t0 = time.perf_counter()
    pcg = sf.PCG(M)
    setup = time.perf_counter() - t0
    b = sf.gen_vector(M.n, 7)
    pcg.solve(b, rtol=1e-10, maxit=1000)  # warm-up
    x, it, rr, ms = pcg.solve(b, rtol=1e-10, maxit=1000)
    out["pcg_config2"] = {"workload": "PCG + IC0 on the config-2 matrix (7-pt 64^3, diag 6.01), "
                                      "rtol 1e-10, b = gen_vector(n, 7)",
                          "iterations": it, "relres": rr, "solve_ms": ms,
                          "ms_per_iteration": ms / max(it, 1), "setup_s": setup}
    pcg.close()
    return out


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU fused executor
# ---------------------------------------------------------------------------
def run_reference(args, D: Dist):
    if D.rank != 0:
        return None
    from oracle.oracle import Reference
    cfg = args.config
    if not Reference.available():
        return {"impl": "reference", "unavailable": "oracle/_ref/libsfref.so not built"}
    ref = Reference()
    T = cpu_threads()
    warm = max(args.warmup, 1)
    if cfg == 5:
        # BASELINE's whole batch of 8 every step, like our arm's global batch
        nsys = 8 if args.systems_per_gpu is None else args.systems_per_gpu * D.world
        M, vals, vin = ref_inputs(ref, 5, args.size, nsys, 0)
        r = RefConfig5(ref, M, vals, vin, nsys, T)
        for _ in range(warm):
            r.step()
        times = [r.step() for _ in range(args.steps)]
        mean_s = float(np.mean(times))
        value = nsys / mean_s
        combo, insp, nsp = 8, r.inspector_s, None
        sample = (f"the whole batch of {nsys} systems per step, each a fwd L then bwd L^T solve "
                  f"on the reference's parallel executor (execute_unfused, LBC schedules, T={T}; "
                  "the reference has no fwd->bwd pair), sum of executor wall times; "
                  f"{args.steps} steps after {warm} warm-ups; schedules built once "
                  f"({insp:.1f}s, excluded)")
        cfgd = workload_config(5, 8, M.n, M.nnz, lower_nnz(M), nsys // D.world, D.world)
    else:
        M, _, vin = ref_inputs(ref, cfg, args.size)
        r = reference_fused(cfg, M, vin, T, warmups=warm, repeats=args.steps)
        mean_s = float(np.mean(r["times"]))
        value = 1.0 / mean_s
        combo, insp, nsp = r["combo"], r["inspector_s"], r["s_partitions"]
        sample = (f"reference execute_fused, T={T} host threads, 1 execution per step "
                  f"({args.steps} steps after {warm} warm-ups; msp inspector {insp:.1f}s excluded)")
        cfgd = workload_config(cfg, combo, M.n, M.nnz, lower_nnz(M), 1, D.world)
    assert "paper_2111_12238_b200" not in sys.modules, "the reference arm must not load our package"
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": D.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_s * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfgd,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": T, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "inspector_s": insp, "s_partitions": nsp, "package_loaded": False,
    }


class _Solo(Dist):
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = 0
        self.local = 0
        self.pg = None

    def barrier(self):
        pass

    def max(self, x):
        return x

    def close(self):
        pass


def spawn_ranks(n: int) -> int:
    """--gpus N without a torchrun environment: launch the N ranks here
    (torch.distributed.run on 127.0.0.1, one process per GPU).  Rank 0
    prints the JSON line."""
    import socket
    import subprocess
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=5, choices=(1, 2, 3, 4, 5))
    ap.add_argument("--mode", choices=("fwdbwd", "fwdfwd"), default="fwdbwd")
    ap.add_argument("--systems-per-gpu", type=int, default=None,
                    help="config 5: systems on every GPU (weak scaling); default: the batch "
                         "of 8 split over the GPUs")
    ap.add_argument("--size", type=int, default=None, help="grid side / n override (testing)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--shard-spmv", action="store_true",
                    help="config 1 only: solve on rank 0, SpMV rows sharded over ranks")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        ap.error(f"--gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}")
    if args.impl == "reference" and int(os.environ.get("RANK", "0")) != 0:
        return  # the reference arm runs on rank 0 only
    D = Dist() if args.impl == "ours" else _Solo()
    try:
        if args.impl == "reference":
            line = run_reference(args, D)
        elif args.shard_spmv:
            if args.config != 1:
                raise SystemExit("--shard-spmv applies to --config 1")
            line = run_sharded(args, D)
        else:
            line = run_ours(args, D)
        if D.rank == 0 and line is not None:
            print(json.dumps(line), flush=True)
    finally:
        D.close()


if __name__ == "__main__":
    main()
