"""Per-solve timeline of k_branch_al (diagnostic; needs a -DUCAC_PROF build):
python tools/al_timeline.py [iterations]  -> distribution of solve durations, per-warp spans."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_13145_b200 import inputs, ucac  # noqa: E402


def main(iters=10):
    pb, pr = inputs.build_config("pegase2869")
    c = ucac.Context(pb, pr)
    c.iterate(int(iters))
    r0 = c.report()
    c.iterate_timed(1)
    r1 = c.report()
    n = int(r1["al_active"] - r0["al_active"])
    buf = np.zeros(6 << 16, dtype=np.uint64)
    ucac.lib().ucac_debug_prof(buf.ctypes.data_as(C.c_void_p), C.c_size_t(buf.nbytes))
    a = buf[:6 * n].reshape(n, 6).astype(np.int64)
    t0 = a[:, 1].min()
    dur = (a[:, 2] - a[:, 1]) / 1e3
    print(f"{n} AL solves; kernel span {(a[:, 2].max() - t0) / 1e3:.1f} us; start spread {(a[:, 1].max() - t0) / 1e3:.1f} us")
    print("solve duration us: p50 %.1f p90 %.1f p99 %.1f max %.1f" % tuple(np.percentile(dur, [50, 90, 99, 100])))
    print("newton its: p50 %d p90 %d max %d; rounds max %d" % (np.median(a[:, 3]), np.percentile(a[:, 3], 90),
                                                              a[:, 3].max(), a[:, 4].max()))
    warp = a[:, 5] >> 8
    spans = {}
    for w in np.unique(warp):
        m = warp == w
        spans[w] = ((a[m, 2].max() - a[m, 1].min()) / 1e3, int(a[m, 3].max()), int(a[m, 3].mean()), int(m.sum()))
    ws = sorted(spans.items(), key=lambda kv: -kv[1][0])
    print(f"{len(ws)} warps; span us p50 {np.median([v[0] for _, v in ws]):.1f}")
    for w, (sp, mx, mean, cnt) in ws[:8]:
        print(f"  warp {w}: span {sp:.1f} us, lanes {cnt}, newton max {mx} mean {mean}")
    worst = np.argsort(-a[:, 3])[:10]
    print("slowest solves (l, t, newton, rounds):", [(int(a[i, 0]) // pb.T, int(a[i, 0]) % pb.T, int(a[i, 3]), int(a[i, 4]))
                                                   for i in worst])
    # duration per Newton iteration for single solves
    print("us per Newton iteration (solve duration / its): p50 %.2f" % np.median(dur / np.maximum(a[:, 3], 1)))


if __name__ == "__main__":
    main(*sys.argv[1:])
