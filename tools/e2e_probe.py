"""Where the host-API step's time goes beyond the device step (cfg2):
    python tools/e2e_probe.py [--workload cfg2]"""
import argparse
import cProfile
import pstats
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2306_05893_b200.integrator import SimState  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    args = ap.parse_args()
    W = bench.build_workload(args.workload)
    st = W["state"].to_host()
    host = SimState(st.positions, st.velocities, st.accelerations, st.f_int, st.f_ext, st.time)
    dev = W["state"]
    solve, integ = W["solvers"]["ldlt"], W["integ"]
    for _ in range(3):
        integ.compute_step(host, solve)
        integ.compute_step(dev, solve)
    torch.cuda.synchronize()

    def wall(fn, reps=30):
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        return statistics.median(ts)

    out = {"host_step_ms": wall(lambda: integ.compute_step(host, solve)),
           "device_state_step_ms": wall(lambda: integ.compute_step(dev, solve))}
    # host-side enqueue cost alone: the device step without the final wait
    ts = []
    for _ in range(30):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a, b, *_ = integ._assemble_device(integ._flat_dev(dev.positions), integ._flat_dev(dev.velocities),
                                          integ._flat_dev(dev.f_ext))
        solve(a, b)
        ts.append((time.perf_counter() - t0) * 1e3)
        torch.cuda.synchronize()
    out["enqueue_assembly_plus_solve_ms"] = statistics.median(ts)
    print(out)
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(50):
        integ.compute_step(host, solve)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
