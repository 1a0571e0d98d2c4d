#!/usr/bin/env python
"""Benchmark of the per-timestep L-BFGS solver (BASELINE.json metric:
"solver iterations/sec & tet evals/sec (fp64) vs HBM roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One step = one frame (simulate_frame) of the configuration.  BASELINE.json's
metric names no configuration, so the default workload is the largest
configuration that runs on one GPU as a single system: configs[2] (c3:
100x25x25 spline bar, 375 000 tets, 10 L-BFGS iterations per frame).  N > 1:
launched by torch.distributed.run, one process per GPU; c1-c3 do not shard
(independent replicas per rank, "weak"), c4 splits its fixed 1024 instances
across ranks (no data-path collective, "strong"), c5 splits one mesh into
x-slabs (NCCL, "strong").  Timing: CUDA events on the launching stream around
each frame, L2 flushed (256 MiB write) between frames, max over ranks.
`--impl reference` times the CPU oracle port of the reference (oracle/, numpy +
scipy sparse factor) on host threads, one full frame per step (the same
iterations per step as the GPU arm).
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

METRIC = "solver iterations/sec & tet evals/sec (fp64) vs HBM roofline, 1/2/4/8 B200"
UNIT = "iterations/s"
FLUSH_BYTES = 256 << 20


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-graph", action="store_true", help="host-driven body loop (for per-kernel ncu lists)")
    p.add_argument("--slab", action="store_true",
                   help="c5: slab-decomposed frame (one slab per rank; the default for c5 when N > 1)")
    p.add_argument("--fp32", action="store_true",
                   help="the optional fp32 element pass (configs[2] 'optional fp32 run'; fp64 elsewhere)")
    p.add_argument("--coarse", action="store_true",
                   help="c5 slab frame: two-level preconditioner also at N = 1 (always on for N > 1)")
    return p.parse_args()


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed
    region: NVML polled every ~2 ms from a thread (nvidia-smi -lms as fallback)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, {reasons})
        self.proc = None
        self.nvml = None
        self.stop_evt = threading.Event()

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            bits = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.nvml = pynvml

            def poll():
                while not self.stop_evt.is_set():
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((float(sm), float(mx), {self.NAMES[i] for i, b in enumerate(bits) if rs & b}))
                    time.sleep(0.002)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6 and parts[0].replace(".", "").isdigit():
                self.rows.append((float(parts[0]), float(parts[1]) if parts[1].replace(".", "").isdigit() else None,
                                  {self.NAMES[i] for i in range(4) if parts[2 + i].lower() == "active"}))

    def stop(self):
        if self.nvml is not None:
            self.stop_evt.set()
            self.t.join(timeout=2)
            src = "nvml"
        elif self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)
            src = "nvidia-smi"
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock source"], "samples": 0}
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0, "source": src}
        sm = [r[0] for r in rows]
        mx = [r[1] for r in rows if r[1]]
        reasons = sorted(set().union(*[r[2] for r in rows]))
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "source": src}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def ncu_traffic(workload, kernel):
    """dram bytes per launch of `kernel` on `workload` from the committed ncu
    --set full summaries, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(workload, {}).get(kernel)
    except (OSError, ValueError, AttributeError):
        return None


FP64_PEAK_TFLOPS = 34.37  # DFMA microbenchmark on this pool's B200 (tools/probe_device.cu, profiles/r01_device_probe.txt)
# fp64 flops per tet eval (2 DFMA + DMUL + DADD) from ncu sass counters of the per-tet kernel
# (smsp__sass_thread_inst_executed_op_d{fma,mul,add}_pred_on.sum / tets), per workload because the
# material (and the SVD sweep count of the state) changes the count: profiles/r0*_fp64_flops*.txt
FLOPS_PER_TET = {
    "c1": (1478.0, "ncu sass counters, c1 Neo-Hookean after 3 frames (profiles/r02_fp64_flops.txt)"),
    "c2": (1388.0, "ncu sass counters, c2 StVK (profiles/r01_fp64_flops.txt)"),
    "c3": (1533.0, "ncu sass counters, c3 Hermite splines after 3 frames (profiles/r02_fp64_flops.txt)"),
    "c4": (1466.0, "ncu sass counters, c4 1024 x Neo-Hookean after 3 frames (profiles/r02_fp64_flops.txt)"),
    "c5": (1418.0, "ncu sass counters, c5 poly + log material on a 100x25x25 bar (profiles/r02_fp64_flops.txt)"),
}


def tet_fp64(sc, tets, tet_ms):
    """The per-tet kernel against the FP64 roofline (report K1 against
    max(bytes/BW, flops/FP64 peak))."""
    fpt, src = FLOPS_PER_TET.get(sc.name.split("_")[0], (None, None))
    if fpt is None:
        return None
    tf = fpt * tets / (tet_ms * 1e-3) / 1e12
    return {"flops_per_tet": fpt, "achieved_tflops": tf, "peak_tflops": FP64_PEAK_TFLOPS,
            "frac": tf / FP64_PEAK_TFLOPS, "flops_source": src}


def frame_timeline(system, run, stream):
    """Mean in-graph duration (us) per body pass of one traced frame (globaltimer
    stamps written by the kernels themselves, qn_system_timeline): k_grad,
    the solve (k_grad end -> k_eta entry), k_vec and k_tet."""
    import ctypes as C
    from paper_1604_07378_b200 import _lib
    lib = _lib.load()
    passes, kernels = 512, 7  # kTimelinePasses, kTimelineKernels (csrc/qn_common.cuh)
    buf = np.zeros(passes * kernels * 2, dtype=np.uint64)
    try:
        _lib.check(lib.qn_system_set_timeline(system._h, 1))
        run.step(stream=stream.cuda_stream)
        _lib.check(lib.qn_system_timeline(system._h, _lib.ptr(buf), C.c_int64(buf.size)))
    finally:
        _lib.check(lib.qn_system_set_timeline(system._h, 0))
    t = buf.reshape(passes, kernels, 2).astype(np.int64)
    npass = int((t[:, 3, 1] > 0).sum())
    if npass == 0:
        return None
    full = [p for p in range(npass) if t[p, 0, 1] and t[p, 1, 0]]
    def mean(vals):
        return float(np.mean(vals)) / 1000.0 if len(vals) else None
    return {"passes": npass,
            "grad": mean([t[p, 0, 1] - t[p, 0, 0] for p in full]),
            "solve": mean([t[p, 1, 0] - t[p, 0, 1] for p in full]),
            "tet": mean([t[p, 3, 1] - t[p, 3, 0] for p in range(npass)]),
            "solve_forward": mean([t[p, 4, 1] - t[p, 4, 0] for p in full if t[p, 4, 0] and t[p, 4, 1]]),
            "solve_top": mean([t[p, 6, 1] - t[p, 6, 0] for p in full if t[p, 6, 0] and t[p, 6, 1]]),
            "solve_backward": mean([t[p, 5, 1] - t[p, 5, 0] for p in full if t[p, 5, 0] and t[p, 5, 1]]),
            "frame": (t[npass - 1, 3, 1] - (t[0, 0, 0] or t[0, 3, 0])) / 1000.0}


def scaling_of(workload):
    """c4's 1024 instances and c5's one mesh are fixed totals split over the ranks
    (strong); c1-c3 run one replica per rank (weak)."""
    return "strong" if workload in ("c4", "c5") else "weak"


def build_scene(name, rank, world):
    from paper_1604_07378_b200 import scenes
    sc = scenes.CONFIGS[name]()
    if name == "c4":  # shard independent instances across ranks (no collective on the data path)
        from paper_1604_07378_b200.parallel import shard_instances
        lo, hi = shard_instances(len(sc.batch_materials), world, rank)
        sc.batch_materials = sc.batch_materials[lo:hi]
        sc.q_l, sc.q_prev = sc.q_l[lo:hi], sc.q_prev[lo:hi]
    return sc


def build_system(sc):
    import paper_1604_07378_b200 as Q
    from paper_1604_07378_b200.materials import from_spec
    mesh = Q.TetMesh(sc.verts, sc.tets, sc.density)
    if sc.batch:
        return Q.build_batch_system(mesh, [from_spec(s) for s in sc.batch_materials], h=sc.h, gravity=sc.gravity,
                                    fixed=sc.fixed)
    solver = "amg" if sc.name.startswith("c5") else "direct"  # configs[4]: (AMG-)PCG to 1e-10 (BASELINE.json)
    return Q.build_system(mesh, from_spec(sc.material), h=sc.h, gravity=sc.gravity, fixed=sc.fixed, solver=solver,
                          pcg_tol=1e-10)


def cpu_oracle_rate(sc, iterations, frames=1, threads=1):
    """Reference CPU path (oracle port, sparse factor restatement) iterations/s."""
    import oracle.qnsim_oracle as O
    from tests.helpers import oracle_material
    O.set_threads(threads)
    spec = sc.batch_materials[0] if sc.batch else sc.material
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(spec), sc.h, sc.gravity, sc.fixed)
    q_l = np.array(sc.q_l[0] if sc.batch else sc.q_l)
    q_prev = np.array(sc.q_prev[0] if sc.batch else sc.q_prev)
    t = time.perf_counter()
    for _ in range(frames):
        x, _, _ = O.simulate_frame(osys, q_l, q_prev, iterations=iterations, m=sc.m)
        q_prev, q_l = q_l, x
    dt = time.perf_counter() - t
    return iterations * frames / dt, dt


def arm_config(workload, sc, tets, verts, instances, world):
    """`config` of the JSON line: the workload, shared by the GPU arm and the `--impl reference` arm."""
    return {"workload": workload, "tets": tets, "verts": verts, "instances": instances,
            "iterations_per_step": sc.iterations, "m": sc.m,
            "l2": "flushed between steps (256 MiB write)",
            "parallelism": "replicas" if not sc.batch else f"instances/{world} per rank"}


def run_reference(args, world, rank):
    if rank != 0:
        return
    from paper_1604_07378_b200 import scenes
    if args.config == "c5":  # the oracle's sparse LU of a 12 M-dof A_free does not fit a bounded host run
        emit({"impl": "reference", "metric": METRIC, "unit": UNIT, "n_gpus": world, "value": None,
                          "unavailable": "configs[4]: the CPU oracle factors A_free (12 M dofs); not a bounded "
                                         "host run (DESIGN.md section 6)"})
        return
    sc = scenes.CONFIGS[args.config]()
    threads = os.cpu_count() or 1
    import oracle.qnsim_oracle as O
    from tests.helpers import oracle_material
    O.set_threads(threads)
    spec = sc.batch_materials[0] if sc.batch else sc.material
    osys = O.build(sc.verts, sc.tets, sc.density, oracle_material(spec), sc.h, sc.gravity, sc.fixed)
    q_l = np.array(sc.q_l[0] if sc.batch else sc.q_l)
    q_prev = np.array(sc.q_prev[0] if sc.batch else sc.q_prev)
    its = sc.iterations  # one whole frame per step: the GPU arm's iterations_per_step
    warm = min(args.warmup, 1)  # host code has no JIT / cache warm-up beyond the first frame
    times = []
    for k in range(warm + args.steps):
        t = time.perf_counter()
        x, _, _ = O.simulate_frame(osys, q_l, q_prev, iterations=its, m=sc.m)
        dt = time.perf_counter() - t
        q_prev, q_l = q_l, x
        if k >= warm:
            times.append(dt)
    total = sum(times)
    value = its * args.steps / total  # (instance-)iterations per second on the host
    sample = (f"{args.steps} consecutive {args.config} frames x {its} L-BFGS iterations from the scene's initial "
              f"state after {warm} untimed frame(s) (oracle port, sparse LU factor, {threads} element-pass threads)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / args.steps,
            "higher_is_better": True, "scaling": scaling_of(args.config), "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            # the GPU arm's config, key for key (the driver compares the two arms' configs); the host run
            # times ONE instance of a batched workload (see `sample`)
            "config": arm_config(args.config, sc, int(sc.tets.shape[0]), int(sc.verts.shape[0]),
                                 len(sc.batch_materials) if sc.batch else 1, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def run_ours(args, world, rank, local):
    import torch
    import paper_1604_07378_b200 as Q
    from paper_1604_07378_b200 import _lib

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sc = build_scene(args.config, rank, world)
    n_inst = max(1, sc.batch)
    t_build = time.perf_counter()
    system = build_system(sc)
    if args.fp32:
        system.set_precision("fp32")
    t_build = time.perf_counter() - t_build
    cfg = Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m)
    st0 = Q.SimState(q_l=sc.q_l, q_prev=sc.q_prev)
    if args.no_graph:
        system.set_graph_mode(False)
    run = Q.ResidentRun(system, st0, cfg)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    for _ in range(args.warmup):
        run.step(stream=sptr)
    # ---- timed region: K frames, device-resident state, L2 flushed between frames ----
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    passes = cg_iters = 0
    l0 = _lib.launch_count()
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record(stream)
        run.step(stream=sptr)
        ev[k][1].record(stream)
        passes += run.last_passes
        cg_iters += run.last_cg_iterations
    torch.cuda.synchronize()
    launches = _lib.launch_count() - l0
    clk = clocks.stop()
    ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(ms)
    if world > 1:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    its_per_step = sc.iterations * n_inst
    value = world * its_per_step * args.steps / (total_ms / 1000.0)
    tet_evals = world * passes * sc.tets.shape[0] * n_inst / (total_ms / 1000.0)

    # ---- roofline of the hot kernels (stand-alone CUDA-event timing, same stream,
    #      every instance) + their live in-graph durations from one traced frame ----
    hbm, peak_kind = peaks()
    info = system.factor_info()
    m, n = sc.tets.shape[0], sc.verts.shape[0]
    tet_ms = system.time_kernel("tet", reps=20, stream=sptr)
    # idx + Dm^-1 + vol (96 B/tet) are shared by all instances of a batch (one mesh,
    # qn_kernels.cuh: no instance term); forces (96 B) and the x gather (24 n/m)
    # are per instance
    tet_bytes = 96.0 * m + (96.0 + 24.0 * n / m) * m * n_inst
    per_frame = total_ms / args.steps
    share_tet = tet_ms * passes / args.steps / per_frame
    batched = info.get("nbatch", 1) > 1
    if "nnz_l" in info:
        solve_ms = system.time_kernel("solve", reps=20, stream=sptr)
        # per instance: L of the sparse sweeps read twice (forward, backward), the
        # dense top's symmetric S^-1 read once (half: K (K + 1) / 2), rhs/y/x/u vectors
        K = info.get("dense_top", 0) or 0
        solve_bytes = (2 * 8.0 * info.get("nnz_l_sparse", info["nnz_l"]) + 8.0 * K * (K + 1) / 2
                       + 5 * 24.0 * info["n"]) * n_inst
        share_solve = solve_ms * sc.iterations / per_frame
    else:  # PCG / AMG system: the CG SpMV and (AMG) the V-cycle, shares from CG iterations per step
        solve_ms = system.time_kernel("spmv", reps=20, stream=sptr)
        nnz_a = system.a_nnz
        # the CG's own SpMV kernel (p = z + beta p_old formed in the neighbour loads): matrix once (fp64
        # value + int32 column), p_old and z read once (z: fp32 rows of 16 B after the AMG cycle, else
        # r and dinv), p and q written
        # AMG (recurrence form, k_pcg_spmv_rec): z gathered, p_old and q_old read, p and q written
        if info.get("solver") == "amg":
            solve_bytes = 12.0 * nnz_a + (16.0 + 48.0 + 48.0) * system.n_free
        else:
            solve_bytes = 12.0 * nnz_a + (24.0 + 32.0 + 48.0) * system.n_free
        share_solve = 0.0
    live = frame_timeline(system, run, stream)
    cg_per_step = cg_iters / args.steps
    vcyc = None
    if "nnz_l" not in info:
        share_solve = solve_ms * cg_per_step / per_frame  # the SpMV's share of the step
        amg = info if info.get("solver") == "amg" else None
        if amg:
            vc_ms = system.time_kernel("vcycle", reps=10, stream=sptr)
            rows, nA, nP, nR = amg["rows"], amg["nnz_A"], amg["nnz_P"], amg["nnz_R"]
            # per level l < coarsest: A twice (residual, post-smoothing), P and R once, fp32 values +
            # int32 columns = 8 B per entry; the cycle's vectors are fp32 rows of 16 B (level 0 reads
            # the fp64 CG residual and writes z in fp64, 24 B per row): residual (x gathered, b read,
            # r written), restriction (r gathered; b, x written and dinv read on the coarse level),
            # prolongation (coarse t gathered, x read + written), post-smoothing (x gathered, b, dinv
            # read, t written), level-0 pre-smoothing (b, dinv read, x written); coarsest: dense fp32
            # inverse (nc^2) + its vectors
            vb = 0.0
            for l in range(len(rows) - 1):
                bt = 24.0 if l == 0 else 16.0
                vb += 8.0 * (2 * nA[l] + nP[l] + nR[l])
                vb += rows[l] * ((16 + bt + 16) + 16 + 32 + (16 + bt + 8 + bt)) + rows[l + 1] * (32 + 8 + 16)
            vb += rows[0] * (24 + 8 + 16)
            vb += 4.0 * rows[-1] ** 2 + 32.0 * rows[-1]
            vcyc = {"ms": vc_ms, "algorithmic_bytes": vb, "GBps": vb / vc_ms / 1e6,
                    "share": vc_ms * cg_per_step / per_frame, "kernels": "k_amg_presmooth, k_amg_residual/"
                    "restrict/coarse/prolong/smooth over the levels", "levels": len(rows)}
    cands = {"tet": (share_tet, tet_ms, tet_bytes), "solve": (share_solve, solve_ms, solve_bytes)}
    if vcyc:
        cands["vcycle"] = (vcyc["share"], vcyc["ms"], vcyc["algorithmic_bytes"])
    dom = max(cands, key=lambda k: cands[k][0])
    _, dms, dbytes = cands[dom]
    achieved = dbytes / (dms / 1000.0) / 1e9
    solve_name = ("sptrsv_batch (level-parallel, CTA per instance)" if batched else
                  ("sptrsv_forward + top (symmetric S^-1) + backward" if info.get("dense_top") else
                   "sptrsv_forward+backward") if "nnz_l" in info else "k_pcg_spmv (CG SpMV, SELL-32 fp64)")
    names = {"tet": "k_tet (per-tet F/SVD/VL/PK1)", "solve": solve_name,
             "vcycle": "AMG V(1,1) cycle (k_amg_presmooth/residual/restrict/coarse/prolong/smooth, all levels)"}
    roof = {"bound": "hbm", "kernel": names[dom],
            "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm, "peak_kind": peak_kind,
            "traffic": ncu_traffic(args.config, dom), "algorithmic_bytes": dbytes, "launch_ms": dms,
            "share_of_step": cands[dom][0],
            "other": {"tet_ms": tet_ms, "tet_GBps": tet_bytes / tet_ms / 1e6, "tet_share": share_tet,
                      "tet_fp64": tet_fp64(sc, m * n_inst, tet_ms),
                      "solve_ms": solve_ms if solve_bytes else None,
                      "solve_GBps": solve_bytes / solve_ms / 1e6 if solve_bytes else None,
                      "solve_share": share_solve, "vcycle": vcyc, "in_graph_us_per_pass": live}}

    # ---- e2e through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        # page-locked host buffers, rotated so a frame never writes the arrays it reads
        shape = np.asarray(sc.q_l).shape
        keep = [torch.empty(shape, dtype=torch.float64, pin_memory=True) for _ in range(4)]
        host = [k.numpy() for k in keep]
        host[0][...] = sc.q_l
        host[1][...] = sc.q_prev
        st = Q.SimState(q_l=host[0], q_prev=host[1])
        y_host = host[3]
        slot = 2

        def frame(st, slot):
            out = Q.SimState(q_l=host[slot], q_prev=st.q_l, y=y_host)
            nxt, _ = Q.simulate_frame(system, st, cfg, out=out)
            used = {id(nxt.q_l), id(nxt.q_prev)}
            free = next(i for i in range(3) if id(host[i]) not in used)
            return nxt, free

        for _ in range(min(args.warmup, 2)):
            st, slot = frame(st, slot)
        if world > 1:
            torch.distributed.barrier()
        t = time.perf_counter()
        for _ in range(args.steps):
            st, slot = frame(st, slot)
        dt = time.perf_counter() - t
        if world > 1:
            tt = torch.tensor([dt], device="cuda", dtype=torch.float64)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            dt = float(tt.item())
        vec = n_inst * n * 3 * 8
        rec_bytes = n_inst * (cfg.iterations * (8 * 3 + 4) + 8 + 4)
        e2e = {"value": world * its_per_step * args.steps / dt, "unit": UNIT, "h2d_bytes_per_step": 2 * vec,
               "d2h_bytes_per_step": 2 * vec + rec_bytes}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and "nnz_l" not in info:
        # configs[4]: the oracle's sparse LU of the 12 M-dof A_free is infeasible on the host
        cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": "not run: the CPU oracle factors A_free (12 M dofs at configs[4]); DESIGN.md section 6"}
    elif rank == 0 and world == 1 and not args.no_cpu:
        cpu_its = 8 if m > 10000 else sc.iterations
        rate, dt = cpu_oracle_rate(sc, cpu_its, frames=1 if m > 10000 else 5)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{cpu_its if m > 10000 else 5 * cpu_its} L-BFGS iterations of {args.config} from its "
                         f"initial state, 1 thread ({dt:.1f} s)"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": per_frame, "higher_is_better": True,
                "scaling": scaling_of(args.config), "vs_baseline": None,
                "dtype": "f32 element pass, f64 elsewhere" if args.fp32 else "f64",
                "data": "synthetic",
                "config": arm_config(args.config, sc, int(m), int(n), n_inst * world, world),
                "tet_evals_per_s": tet_evals, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "clocks": clk, "gpu_launches": launches,
                "factor": ({"nnz_l": info["nnz_l"], "nnz_l_sparse": info.get("nnz_l_sparse"),
                            "supernodes": info["n_supernodes"],
                            "depth": info["tree_depth"], "factor_s": info["factor_seconds"],
                            "dense_top": info.get("dense_top")} if "nnz_l" in info else info),
                "build_s": t_build, "build_phases_s": getattr(system, "build_times", None),
                "passes_per_step": passes / args.steps}
        if cg_iters:
            line["cg_iterations_per_step"] = cg_iters / args.steps
        emit(line)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_slab(args, world, rank, local):
    """configs[4] as one mesh split into `world` x-slabs, one per GPU (SURVEY
    §8e): per-rank stage kernels, NCCL all-gathers of the partial sums, NCCL
    send/recv of the boundary planes (paper_1604_07378_b200/slab.py).  Total
    work is fixed, so the scaling is strong; value = L-BFGS iterations of the
    one mesh per second (max over ranks)."""
    import torch
    import torch.distributed as dist
    import paper_1604_07378_b200 as Q
    from paper_1604_07378_b200 import _lib, scenes, slab
    from paper_1604_07378_b200.materials import from_spec
    from paper_1604_07378_b200.mesh import TetMesh, lumped_masses

    torch.cuda.set_device(local)
    dist.init_process_group("nccl", init_method=None if world > 1 else "tcp://127.0.0.1:%d" % _free_port(),
                            rank=rank, world_size=world, device_id=torch.device("cuda", local))
    grid = (400, 100, 100)
    iterations, m_hist = 10, 5
    t_build = time.perf_counter()
    verts, spec, fixed = scenes.c5_vertices(grid=grid)
    lay = slab.slab_layout(grid, world, rank)
    size = tuple(scenes.SPACING * g for g in grid)
    tets = slab.local_tets_generated(lay, size)
    vl = verts[lay.v0: lay.v0 + lay.n]
    rk = slab.SlabRank(lay, vl, tets, from_spec(spec), fixed, scenes.H, scenes.GRAVITY, scenes.DENSITY,
                       solver="amg", pcg_tol=1e-10)
    rk.set_state(vl, vl)
    mm = torch.tensor([float(lumped_masses(TetMesh(vl, tets, scenes.DENSITY))[lay.own_lo:lay.own_hi].max())],
                      dtype=torch.float64, device="cuda")
    dist.all_reduce(mm, op=dist.ReduceOp.MAX)
    bbox = float(np.linalg.norm(verts.max(axis=0) - verts.min(axis=0)))
    t_build = time.perf_counter() - t_build
    cfg = Q.SolverConfig(kind="lbfgs", iterations=iterations, m=m_hist)
    comm = slab.NcclComm(rk)
    t_coarse = time.perf_counter()
    if world > 1 or args.coarse:  # two-level preconditioner: per-slab AMG + geometric coarse grid (slab.setup_coarse)
        slab.setup_coarse(comm, grid)
    t_coarse = time.perf_counter() - t_coarse
    run = slab.SlabRun(comm, cfg, scenes.H, slab.grad_tolerance(bbox, float(mm.item()), scenes.H))
    stream = torch.cuda.current_stream()
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    for _ in range(args.warmup):
        run.step()
    dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    evals = 0
    cg0 = run.cg_iterations
    l0 = _lib.launch_count()
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record(stream)
        rec = run.step()
        ev[k][1].record(stream)
        evals += 1 + sum(rec.ls_trials)
    torch.cuda.synchronize()
    launches = _lib.launch_count() - l0
    clk = clocks.stop()
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    per_frame = total_ms / args.steps
    m_all = 6 * grid[0] * grid[1] * grid[2]
    n_all = verts.shape[0]
    value = iterations * args.steps / (total_ms / 1000.0)
    # roofline: the CG SpMV of this rank's owned block (the local system's A_oo, same rows)
    hbm, peak_kind = peaks()
    spmv_ms = rk.system.time_kernel("spmv", reps=20, stream=stream.cuda_stream)
    spmv_bytes = 12.0 * rk.system.a_nnz + 2 * 24.0 * rk.system.n_free
    achieved = spmv_bytes / (spmv_ms / 1000.0) / 1e9
    cg_per_step = (run.cg_iterations - cg0) / args.steps
    roof = {"bound": "hbm", "kernel": "CG SpMV of the rank's owned block (SELL-32 fp64)", "achieved": achieved,
            "peak": hbm, "unit": "GB/s", "frac": achieved / hbm, "peak_kind": peak_kind, "traffic": None,
            "algorithmic_bytes": spmv_bytes, "launch_ms": spmv_ms,
            "share_of_step": None}
    # e2e: state from / positions to page-locked host buffers every frame
    e2e = None
    if not args.no_e2e:
        hq = torch.empty(lay.n * 3, dtype=torch.float64, pin_memory=True)
        hp = torch.empty(lay.n * 3, dtype=torch.float64, pin_memory=True)
        hx = torch.empty((lay.own_hi - lay.own_lo) * 3, dtype=torch.float64, pin_memory=True)
        hq.copy_(rk.buf[slab.QL])
        hp.copy_(rk.buf[slab.QPREV])
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            rk.buf[slab.QL].copy_(hq, non_blocking=True)
            rk.buf[slab.QPREV].copy_(hp, non_blocking=True)
            run.step()
            hx.copy_(rk.buf[slab.QL][lay.own_lo * 3: lay.own_hi * 3], non_blocking=True)
            torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], device="cuda", dtype=torch.float64)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": iterations * args.steps / float(dt.item()), "unit": UNIT,
               "h2d_bytes_per_step": 2 * lay.n * 24 * world, "d2h_bytes_per_step": n_all * 24}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": per_frame, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": "c5", "engine": "slab", "tets": m_all, "verts": n_all,
                           "iterations_per_step": iterations, "m": m_hist, "slabs": world,
                           "l2": "flushed between steps (256 MiB write)", "parallelism": f"x-slabs/{world}",
                           "preconditioner": "per-slab AMG V(1,1) + geometric coarse grid (additive two-level)"
                           if (world > 1 or args.coarse) else "AMG V(1,1)"},
                "tet_evals_per_s": evals * m_all / (total_ms / 1000.0), "roofline": roof, "cpu_baseline": None,
                "e2e": e2e, "clocks": clk, "gpu_launches": launches, "build_s": t_build, "coarse_setup_s": t_coarse,
                "cg_iterations_per_step": cg_per_step}
        emit(line)
    dist.destroy_process_group()


def _free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


_OUT = sys.stdout


def emit(line):
    """The contract's one JSON line, on the real stdout."""
    print(json.dumps(line), file=_OUT, flush=True)


def _private_stdout():
    """Native libraries print to fd 1 (the GPU boxes set NCCL_DEBUG=VERSION, so
    NCCL's banner lands there at communicator creation): fd 1 becomes stderr and
    the JSON line goes through a private duplicate of the original stdout."""
    global _OUT
    sys.stdout.flush()
    fd = os.dup(1)
    os.dup2(2, 1)
    _OUT = os.fdopen(fd, "w", buffering=1)


def main():
    _private_stdout()
    args = parse()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    elif args.config == "c5" and (world > 1 or args.slab):
        run_slab(args, world, rank, local)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
