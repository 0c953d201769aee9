"""One plugin-path pass (BenchWorkload: stage + correlate_batch of 500,000 random
offsets, bench.hpp:65-118) inside a cudaProfilerStart/Stop window, for ncu
--profile-from-start off (k_correlate's launch list and --set full capture).
Not collected by pytest."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2508_06672_b200 as b2  # noqa: E402


def main():
    y1, y2, off = bench.build_workload(bench.PLUGIN_POINTS, bench.PLUGIN_SAMPLES, 5e6, 1)
    be = b2.make_backend("b200", 1)
    c1, c2 = b2.BasebandCapture(y1, 5e6), b2.BasebandCapture(y2, 5e6)
    out = np.zeros(len(off))
    be.stage(c1, c2).correlate_batch(off, out)  # warm-up
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    be.stage(c1, c2).correlate_batch(off, out)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("plugin pass", float(out.sum()))


if __name__ == "__main__":
    main()
