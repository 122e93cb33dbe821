"""Per-CTA %globaltimer timeline of two consecutive launches of one bench.py op.

Same capture as tools/floor_timeline.py (a CUDA graph of back-to-back launches with
PDL edges, one trace buffer per launch), but instead of medians over launches it
prints, for one launch k+1 of the middle of the sequence, every CTA's milestones
relative to the last exit of launch k, grouped by the number of tiles the CTA ran:
  entry      the CTA started (negative: while launch k was still running)
  pdl        griddepcontrol.wait returned in the producer
  full       first operand stage landed
  tfull      first accumulator published
  stores     all TMA stores complete
  exit       the CTA ended
Usage: python tools/cta_timeline.py OP [launch_index]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2207_04296_b200 as tb  # noqa: E402


def capture(op, launches=8):
    dev = torch.device("cuda:0")
    L = tb.lib()
    L.tir_b200_debug_set_trace.argtypes = [ctypes.c_void_p]
    r = bench.OpRunner(op, dev)
    bufs = [torch.zeros(16384, dtype=torch.int64, device=dev) for _ in range(launches)]
    for i in range(3):
        r.step(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="relaxed"):
        for i in range(launches):
            L.tir_b200_debug_set_trace(bufs[i].data_ptr())
            r.step(i)
    L.tir_b200_debug_set_trace(None)
    for _ in range(3):
        for b in bufs:
            b.zero_()
        g.replay()
    torch.cuda.synchronize()
    out = []
    for b in bufs:
        ev = b[8192:8192 + 8 * 256].view(256, 8)[:, :8].cpu().tolist()
        cta = b[2048:2048 + 4 * 1024].view(1024, 4).cpu().tolist()
        xs = b[10240:10240 + 8 * 256].view(256, 8).cpu().tolist()
        out.append(([e + x for e, x in zip(ev, xs)], cta, b[:2048].cpu().tolist()))
    return out


def main():
    op = sys.argv[1] if len(sys.argv) > 1 else "C2D"
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    tl = capture(op)
    prev_ev = tl[k - 1][0]
    ev, cta, clk = tl[k]
    prev_exit = max(e[5] for e in prev_ev if e[0] > 0)
    rows = []
    for b, e in enumerate(ev):
        if e[0] == 0:
            continue
        tiles = cta[b][3] if b < len(cta) else -1
        smid = cta[b][2] if b < len(cta) else -1
        rows.append((tiles, [x - prev_exit if x else None for x in e], smid, b))
    print(f"op {op} launch {k}: {len(rows)} traced CTAs; times in ns relative to launch {k-1}'s last exit")
    # x0..x7: split-K combine (igemm cluster_reduce): x0 entry, x1 first cluster sync passed,
    # x2 tile coordinates read, x3 final sync passed; x4 partial written; x5 kernel-end
    # barrier passed; x6 combine setup done (PDL wait passed); x7 last remote read consumed
    names = ["entry", "pdl", "full", "tfull", "stores", "exit", "issue", "preloop",
             "x0", "x1", "x2", "x3", "x4", "x5", "x6", "x7"]
    by = {}
    for t, e, s, b in rows:
        by.setdefault(t, []).append(e)
    for t in sorted(by):
        es = by[t]
        line = [f"tiles={t:3d} n={len(es):3d}"]
        for i, nm in enumerate(names):
            v = sorted(x[i] for x in es if x[i] is not None)
            if v:
                line.append(f"{nm} {v[0]:>7d}/{v[len(v)//2]:>7d}/{v[-1]:>7d}")
        print("  ".join(line))
    # the latest CTAs to pass the wait, and why
    rows.sort(key=lambda r: r[1][1] or 0)
    print("last 6 CTAs to pass griddepcontrol.wait (block, smid, tiles, entry, pdl, full, exit):")
    for t, e, s, b in rows[-6:]:
        print(f"  block {b:4d} sm {s:4d} tiles {t}  entry {e[0]:>7d} pdl {e[1]:>7d} full {e[2]} exit {e[5]}")
    # previous launch's per-CTA exits (spread of the tail)
    pe = sorted(e[5] - prev_exit for e in prev_ev if e[0] > 0)
    # block 0's SM-clock trace (cycles since its start): producer issue, MMA rounds, epilogue
    t0 = clk[1023]
    if t0:
        prod = [(clk[2 * i] - t0, clk[2 * i + 1] - t0) for i in range(128) if clk[2 * i]]
        mma = [(clk[256 + 2 * i] - t0, clk[257 + 2 * i] - t0) for i in range(128) if clk[256 + 2 * i]]
        epi = [(clk[512 + 2 * i] - t0, clk[513 + 2 * i] - t0) for i in range(64) if clk[512 + 2 * i]]
        print("block 0 (cycles): weights landed", clk[1022] - t0 if clk[1022] else None)
        print("  producer (empty ok, issued):", prod[:12])
        print("  mma (round start, round end):", mma[:12])
        print("  epilogue (tfull ok, done):", epi[:12])
        bld = [tuple(clk[640 + 3 * i + j] - t0 for j in range(3)) for i in range(64) if clk[640 + 3 * i]]
        if bld:
            print("  builder warp (raw ok, A buffer free, A published):", bld[:16])
        pre = [(clk[1024 + 4 * i] - t0, clk[1025 + 4 * i] - t0) for i in range(64) if clk[1024 + 4 * i]]
        if pre:
            print("  MMA plane preamble (start, before A wait) (rowpack):", pre[:12])
        ods = [[clk[832 + 4 * i + j] - t0 for j in range(4) if clk[832 + 4 * i + j]] for i in range(48)
               if clk[832 + 4 * i]]
        if ods:
            print("  MMA per-depth issue done (rowpack):", ods[:16])
    print(f"launch {k-1} exits: first {pe[0]} p10 {pe[len(pe)//10]} median {pe[len(pe)//2]} p90 {pe[9*len(pe)//10]} last {pe[-1]}")


if __name__ == "__main__":
    main()
