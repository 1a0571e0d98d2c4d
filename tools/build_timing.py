"""build_system phase times for a workload (QN_BUILD_VERBOSE / QN_AMG_VERBOSE print the host phases):

    QN_BUILD_VERBOSE=1 QN_AMG_VERBOSE=1 python tools/build_timing.py c5
"""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import bench  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
t = time.time()
sc = bench.build_scene(name, 0, 1)
t_scene = time.time() - t
t = time.time()
system = bench.build_system(sc)
print(f"{name}: scene {t_scene:.2f} s, build_system {time.time() - t:.2f} s, phases {system.build_times}", flush=True)
