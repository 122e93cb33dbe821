"""Per-stage clock64 timeline of CTA 0 of the tcgen05 kernel (debug aid)."""
import ctypes
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch  # noqa: E402

import paper_2207_04296_b200 as tb  # noqa: E402

L = tb.lib()
L.tir_b200_debug_set_trace.argtypes = [ctypes.c_void_p]
dev = torch.device("cuda:0")
buf = torch.zeros(8192, dtype=torch.int64, device=dev)


def show(name, fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    buf.zero_()
    L.tir_b200_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
    fn()
    torch.cuda.synchronize()
    L.tir_b200_debug_set_trace(None)
    t = buf.cpu().tolist()
    t0 = t[1023]
    print(f"== {name} (cycles since CTA start)")
    rows = []
    for it in range(128):
        pe, pi, mf, mc = t[2 * it], t[2 * it + 1], t[256 + 2 * it], t[257 + 2 * it]
        if pe == 0 and mf == 0:
            break
        rows.append((it, pe - t0, pi - t0, mf - t0, mc - t0))
    for r in rows:
        print("stage %3d  prod_wait_done %7d  prod_issued %7d  mma_full %7d  mma_commit %7d" % r)
    for it in range(12):
        w = t[768 + 4 * it: 772 + 4 * it]
        if w[0] == 0:
            break
        continue
        print("stage %2d  after_expect %7d  after_A %7d  before_B %7d  after_B %7d" % (it, *(x - t0 for x in w)))
    ctas = [(t[2048 + 4 * i], t[2049 + 4 * i], t[2050 + 4 * i], t[2051 + 4 * i]) for i in range(1024)]
    ctas = [c for c in ctas if c[0]]
    if ctas:
        t0g = min(c[0] for c in ctas)
        ends = sorted((c[1] - t0g, c[3]) for c in ctas)
        starts = sorted(c[0] - t0g for c in ctas)
        print(f"grid {len(ctas)} CTAs: start spread {starts[0]}..{starts[-1]} ns; end min {ends[0][0]} median {ends[len(ends)//2][0]} max {ends[-1][0]} ns")
        by_tiles = {}
        for e, nt in ends:
            by_tiles.setdefault(nt, []).append(e)
        for nt, es in sorted(by_tiles.items()):
            print(f"  CTAs with {nt} tiles: {len(es)}, end ns min {min(es)} max {max(es)}")
    for i in range(8):
        w = t[1600 + 8 * i: 1607 + 8 * i]
        if w[0] == 0:
            break
        print("halo epi tile %d: ld_issue %7d ld_done %7d epi_done %7d buf_free %7d staged %7d bar2 %7d store_issued+wait1 %7d" % (i, *(x - t0 for x in w)))
    if t[1599]:
        print("epilogue final wait_read done %7d, after __syncthreads %7d" % (t[1599] - t0, t[1598] - t0))
    for i in range(8):
        w = t[1536 + 8 * i: 1543 + 8 * i]
        if w[0] == 0:
            break
        print("tapn epi tile %d: start %7d tfull %7d ld+arrive %7d xbar %7d pre-stage %7d stage-bar %7d stored %7d" % (i, *(x - t0 for x in w)))
    for i in range(64):
        a, b = t[512 + 2 * i], t[513 + 2 * i]
        if a == 0:
            break
        print("tile %2d  epi_start %7d  epi_done %7d" % (i, a - t0, b - t0))


At = torch.randn(128, 64, device=dev).half()
Bt = torch.randn(64, 64, device=dev).half()
show("GMM 128x64x64 (tiny)", lambda: tb.gmm(At, Bt))
A = torch.randn(1024, 1024, device=dev).half()
B = torch.randn(1024, 1024, device=dev).half()
show("GMM 1024", lambda: tb.gmm(A, B))
spec = tb.PAPER_SHAPES["C2D"]
X = torch.randn(*spec.x_shape(), device=dev).half()
W = torch.randn(*spec.w_shape(), device=dev).half()
show("C2D paper", lambda: tb.conv(spec, X, W))
