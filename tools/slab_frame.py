"""Per-stage device time of the slab-decomposed configs[4] frame on one GPU
(CUDA events around every stage and exchange; diagnostics, not a bench).

    python tools/slab_frame.py [--grid 400 100 100] [--world 1] [--frames 1]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1604_07378_b200 as Q  # noqa: E402
from paper_1604_07378_b200 import scenes, slab  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, nargs=3, default=[400, 100, 100])
    ap.add_argument("--world", type=int, default=1)
    ap.add_argument("--frames", type=int, default=1)
    ap.add_argument("--check", type=int, default=4)
    ap.add_argument("--coarse", action="store_true", help="two-level preconditioner (slab.setup_coarse)")
    a = ap.parse_args()
    t = time.perf_counter()
    sc = scenes.c5(grid=tuple(a.grid), frames=a.frames)
    ranks = slab.scene_slabs(sc, a.world)
    comm = slab.EmulatedComm(ranks)
    if a.coarse:
        slab.setup_coarse(comm, sc.grid)
    run = slab.SlabRun(comm, Q.SolverConfig(kind="lbfgs", iterations=sc.iterations, m=sc.m),
                       sc.h, slab.scene_grad_tol(sc), pcg_check=a.check)
    print(f"build {time.perf_counter() - t:.1f} s", flush=True)
    run.step()  # warm-up
    torch.cuda.synchronize()
    run.enable_profile()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cg0 = run.cg_iterations
    e0.record()
    for _ in range(a.frames):
        run.step()
    e1.record()
    tot = run.stage_ms()
    frame = e0.elapsed_time(e1) / a.frames
    print(f"frame {frame:.2f} ms, CG its/frame {(run.cg_iterations - cg0) / a.frames:.1f}")
    acc = 0.0
    for k, (n, ms) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        acc += ms
        print(f"  {k:12s} n={n / a.frames:7.1f}  {ms / a.frames:8.2f} ms  {ms / n * 1000:8.1f} us each")
    print(f"  staged total {acc / a.frames:.2f} ms; gaps {frame - acc / a.frames:.2f} ms")


if __name__ == "__main__":
    main()
