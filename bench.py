"""Benchmark of the tensorized-operator hot path on B200 (contract: see DESIGN.md §Measurement).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--op C2D] [--no-ops] [--no-cpu]

Headline workload (BASELINE.json configs[1]): C2D, ResNet-50 layer shape
N=16, 56x56x64 -> 64, 3x3, stride 1, pad 1, fp16 in / fp32 accumulate / fp32 out,
as one tcgen05 implicit-GEMM launch. A "step" = one operator pass over one
batch. Inputs are resident in HBM; K steps rotate over enough input/output
sets to exceed 2x the 126 MB L2, captured once in a CUDA graph (the launches
are host-bound otherwise) and replayed between CUDA events on the launching
stream. Under torchrun every rank runs its own replica ("replicas only":
single ops do not shard) and the max time over ranks is
reported.

One JSON line on rank 0: the headline metric plus `ops` (the paper's full
single-op sweep measured the same way), `roofline`, `cpu_baseline`, `e2e`
(synchronous host-buffer C-ABI call: H2D + kernel + D2H), `clocks` and
`gpu_launches`.

--impl reference times the reference's own CPU implementation of the path —
tir::run from /root/reference/proj (built into oracle/_ref by oracle/Makefile)
on the host cores, rank 0 only, each step a bounded slice of the same C2D
workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HEADLINE = "C2D"
L2_BYTES = 126 * 1024 * 1024
METRIC = "per-op TFLOPS & % of B200 fp16 tensor peak (DEP: HBM GB/s) vs host-CPU ref"
SPEC_TC_PEAK_TFLOPS = 2250.0


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "fallback"}


# ----------------------------------------------------------------------------- dist

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(n: int) -> None:
    """`bench.py --gpus N` outside torchrun: re-execute this command under
    torch.distributed.run with N ranks (one process per GPU, 127.0.0.1
    rendezvous), exactly as the driver launches it; returns only on failure."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__),
           *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def init_dist(world, backend):
    import torch.distributed as dist

    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return dist if world > 1 else None


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms",
                 "100", "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- workloads

# Extra tensor-bound shapes of SURVEY §8(d) (reported in `ops`, not the headline).
EXTRA_SHAPES = {
    "GMM8K": (8192, 8192, 8192),                     # peak demo
    "C2D_L3": dict(op="C2D", n=16, in_dhw=(1, 14, 14), ci=256, co=256, k=(1, 3, 3), p=(0, 1, 1)),
    "FLOOR": (128, 64, 64),                          # one-CTA GEMM: the per-launch floor
}
# The MobileNet-V2 depthwise layers (BASELINE configs[3]), all 3x3 p1, N = 16.
DEP_SHAPES = {"DEP": (112, 32, 1), "DEP_112c96s2": (112, 96, 2), "DEP_56c144s1": (56, 144, 1),
              "DEP_56c144s2": (56, 144, 2), "DEP_28c192s1": (28, 192, 1), "DEP_28c192s2": (28, 192, 2),
              "DEP_14c384s1": (14, 384, 1), "DEP_14c576s1": (14, 576, 1), "DEP_14c576s2": (14, 576, 2),
              "DEP_7c960s1": (7, 960, 1)}
for _n, (_hw, _c, _s) in DEP_SHAPES.items():
    if _n != "DEP":
        EXTRA_SHAPES[_n] = dict(op="DEP", n=16, in_dhw=(1, _hw, _hw), ci=_c, co=_c, k=(1, 3, 3), s=(1, _s, _s),
                                p=(0, 1, 1), groups=_c)
# the power-heavy long ops (C3D, GMM 8192^3: hundreds of us per launch at the board's power
# cap) run last, so the short ops are not timed in their power / clock aftermath
SWEEP = ["GMM", "C1D", "C2D", "DIL", "GRP", "T2D", *DEP_SHAPES, "C2D_L3", "C3D", "GMM8K"]


def gmm_shape(name):
    import paper_2207_04296_b200 as tb

    return EXTRA_SHAPES[name] if name in EXTRA_SHAPES else tb.GMM_SHAPE


def is_gmm(name):
    return name.startswith("GMM") or name == "FLOOR"


def op_spec(name):
    import paper_2207_04296_b200 as tb

    if is_gmm(name):
        return None
    if name in EXTRA_SHAPES:
        return tb.Conv(**EXTRA_SHAPES[name])
    return tb.PAPER_SHAPES[name]


def op_work(name):
    """(flops, compulsory bytes, roofline bound) of one launch."""
    import paper_2207_04296_b200 as tb

    pk = peaks()
    if is_gmm(name):
        M, N, K = gmm_shape(name)
        flops = 2 * M * N * K
        byts = M * K * 2 + K * N * 2 + M * N * 4
    else:
        spec = op_spec(name)
        flops = 2 * tb.useful_macs(spec)
        byts = tb.compulsory_bytes(spec)
    ridge = pk["bf16_tflops"] * 1e12 / (pk["hbm_gbs"] * 1e9)
    bound = "hbm" if (name.startswith("DEP") or flops / byts < ridge) else "tensor"
    return flops, byts, bound


class OpRunner:
    """Device buffers (rotating sets > 2x L2) + one launch per step."""

    def __init__(self, name, device):
        import torch

        import paper_2207_04296_b200 as tb

        self.name = name
        self.tb = tb
        g = torch.Generator(device=device)
        g.manual_seed(1234)
        if is_gmm(name):
            M, N, K = gmm_shape(name)
            set_bytes = M * K * 2 + K * N * 2 + M * N * 4
            self.sets = int(os.environ.get("BENCH_DIAG_SETS", 0)) or max(2, math.ceil(2 * L2_BYTES / set_bytes))
            self.A = [torch.randn(M, K, device=device, generator=g).half() for _ in range(self.sets)]
            self.B = [torch.randn(K, N, device=device, generator=g).half() for _ in range(self.sets)]
            self.C = [torch.empty(M, N, device=device) for _ in range(self.sets)]
            self.fn = lambda i: tb.gmm(self.A[i], self.B[i], self.C[i])
        else:
            spec = op_spec(name)
            self.spec = spec
            xs, ws, ys = spec.x_shape(), spec.w_shape(), spec.y_shape()
            # every operand rotates (weights too: T2D's 4.2 MB weight panel would
            # otherwise stay L2-resident), > 2x L2 in total
            set_bytes = (math.prod(xs) + math.prod(ws)) * 2 + math.prod(ys) * 4
            # BENCH_DIAG_SETS (diagnostics only, e.g. tools/cta_timeline.py): a fixed set count
            self.sets = int(os.environ.get("BENCH_DIAG_SETS", 0)) or max(2, math.ceil(2 * L2_BYTES / set_bytes))
            self.X = [torch.randn(*xs, device=device, generator=g).half() for _ in range(self.sets)]
            self.W = [torch.randn(*ws, device=device, generator=g).half() for _ in range(self.sets)]
            self.Y = [torch.empty(*ys, device=device) for _ in range(self.sets)]
            self.fn = lambda i: tb.conv(spec, self.X[i], self.W[i], self.Y[i])

    def step(self, i):
        self.fn(i % self.sets)


def time_graph(runner, steps, warmup, dist, sampler_gpu):
    """Returns (elapsed ms for `steps` launches = max over ranks, launches in graph, clocks)."""
    import torch

    tb = runner.tb
    for i in range(warmup):
        runner.step(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    tb.reset_launch_count()
    with torch.cuda.graph(g, capture_error_mode="relaxed"):
        for i in range(steps):
            runner.step(i)
    launches = tb.launch_count()
    g.replay()  # graph warm-up (untimed)
    torch.cuda.synchronize()
    clocks = None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.current_stream()

    def timed():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        return e0.elapsed_time(e1)

    if sampler_gpu is not None:
        with ClockSampler(sampler_gpu) as cs:
            t_end = time.time() + 0.5
            while time.time() < t_end:  # sustained load around the timed region
                g.replay()
            ms = timed()
            t_end = time.time() + 0.5
            while time.time() < t_end:
                g.replay()
            torch.cuda.synchronize()
        clocks = cs.summary()
    else:
        ms = timed()
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    del g
    return ms, launches, clocks


def measure_e2e(name, steps):
    """Synchronous host-buffer C-ABI call (tir_b200_conv_host / gmm_host): pinned fp16
    inputs H2D, kernel, fp32 result D2H, every step. Host wall clock."""
    import numpy as np
    import torch

    import paper_2207_04296_b200 as tb

    rng = np.random.default_rng(7)
    if is_gmm(name):
        M, N, K = gmm_shape(name)
        A = torch.from_numpy(rng.standard_normal((M, K), dtype=np.float32).astype(np.float16)).pin_memory().numpy()
        B = torch.from_numpy(rng.standard_normal((K, N), dtype=np.float32).astype(np.float16)).pin_memory().numpy()
        C = torch.empty((M, N), dtype=torch.float32).pin_memory().numpy()
        fn = lambda: tb.gmm_host(A, B, C)  # noqa: E731
        h2d, d2h = A.nbytes + B.nbytes, C.nbytes
    else:
        spec = op_spec(name)
        X = torch.from_numpy(rng.standard_normal(spec.x_shape(), dtype=np.float32).astype(np.float16)).pin_memory().numpy()
        W = torch.from_numpy(rng.standard_normal(spec.w_shape(), dtype=np.float32).astype(np.float16)).pin_memory().numpy()
        Y = torch.empty(spec.y_shape(), dtype=torch.float32).pin_memory().numpy()
        fn = lambda: tb.conv_host(spec, X, W, Y)  # noqa: E731
        h2d, d2h = X.nbytes + W.nbytes, Y.nbytes
    for _ in range(2):
        fn()
    n = max(3, min(steps, 50))
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    dt = (time.perf_counter() - t0) / n
    flops, _, _ = op_work(name)
    return {"value": round(flops / dt / 1e12, 4), "unit": "TFLOPS", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(dt * 1e3, 4), "steps": n,
            "timing": "host wall clock around the synchronous C-ABI host-buffer call",
            "api": "tir_b200_conv_host" if not is_gmm(name) else "tir_b200_gmm_host"}


def measure_e2e_interp(name, runs=3):
    """The drop-in path exactly as a reference user takes it: the reference's own
    interpreter (tir::run, /root/reference/proj built into oracle/_ref) runs the
    whole-op tensorized program of the headline conv (conv2d_source semantics,
    workloads.h:93-130), and its tensorized block is dispatched through the
    HostKernel adapter (register_conv) -> tir_b200_conv_host_f32 -> B200 kernel.
    Timed on the host clock per complete tir::run, split into view packing
    (TensorView::get_f), the device call (H2D + kernel + D2H) and the write-back
    (TensorView::set_f)."""
    import ctypes

    import numpy as np

    from oracle import ir_gen as G  # the workload program text in the reference grammar

    adapter = os.path.join(ROOT, "paper_2207_04296_b200", "lib", "libtir_b200_adapter.so")
    if not os.path.exists(adapter):
        return {"unavailable": "adapter library not built (needs /root/reference at build time)"}
    L = ctypes.CDLL(adapter)
    f32p = ctypes.POINTER(ctypes.c_float)
    L.tir_b200_adapter_time_run.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(f32p),
                                            f32p, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                            ctypes.POINTER(ctypes.c_double), ctypes.c_char_p, ctypes.c_int]
    spec = op_spec(name)
    ospec = G.ConvSpec(op=spec.op, n=spec.n, in_dhw=spec.in_dhw, ci=spec.ci, co=spec.co, k=spec.k, s=spec.s,
                       p=spec.p, d=spec.d, groups=spec.groups, transposed=spec.transposed)
    rng = np.random.default_rng(11)
    ins = [rng.standard_normal(ospec.x_shape(), dtype=np.float32).astype(np.float16).astype(np.float32),
           rng.standard_normal(ospec.w_shape(), dtype=np.float32).astype(np.float16).astype(np.float32)]
    out = np.zeros(ospec.y_shape(), np.float32)
    arr = (f32p * 2)(*[x.ctypes.data_as(f32p) for x in ins])
    sec = ctypes.c_double(0)
    split = (ctypes.c_double * 3)()
    err = ctypes.create_string_buffer(2048)
    rc = L.tir_b200_adapter_time_run(G.conv_source(ospec).encode(), b"conv", 2, arr, out.ctypes.data_as(f32p),
                                     out.size, runs, ctypes.byref(sec), split, err, len(err))
    if rc != 0:
        return {"error": err.value.decode()[:300]}
    flops, _, _ = op_work(name)
    return {"value": round(flops / sec.value / 1e12, 4), "unit": "TFLOPS",
            "ms_per_step": round(sec.value * 1e3, 3), "runs": runs,
            "split_ms": {"pack_views": round(split[0] * 1e3, 3), "device_call": round(split[1] * 1e3, 3),
                         "unpack_view": round(split[2] * 1e3, 3)},
            "h2d_bytes_per_step": int(sum(x.nbytes for x in ins)),
            "d2h_bytes_per_step": int(out.nbytes),
            "path": "tir::run (reference interpreter) -> whole-op tensorized block (zero init folded: "
                    "overwriting intrinsic) -> HostKernel adapter (register_conv) -> tir_b200_conv_host_f32 "
                    "(f32 views converted to fp16 on the device) -> B200",
            "rest_ms": "tir::run itself: TensorValue allocation / zero-fill and copies of the "
                       "interpreter's input and output tensors"}


TRAFFIC_PROFILE = "r02_ncu_graph_traffic.json"


def traffic_from_profiles(name):
    """Steady-state DRAM read + write bytes per launch of this op, from the committed
    ncu capture of a CUDA graph of consecutive launches on rotating buffers
    (profiles/r02_ncu_graph_traffic.json, tools/ncu_graph_summary.py)."""
    p = os.path.join(ROOT, "profiles", TRAFFIC_PROFILE)
    try:
        with open(p) as f:
            return json.load(f)["ops"][name]["traffic_per_launch"]
    except Exception:
        return None


# ----------------------------------------------------------------------------- networks

NET_BATCH = {"resnet50": 32, "mobilenet_v2": 64, "bert_large": 8}  # per GPU (weak scaling: global = N x this)


def measure_nets(device, world, rank, dist, steps, names):
    """Batch-sharded network forwards: every rank builds the graph of
    its shard of the global batch (replicated weights, no collective), captures it
    in a CUDA graph and replays it `steps` times between CUDA events; images/s =
    global batch x steps / max-over-ranks time."""
    import torch

    from paper_2207_04296_b200 import nets

    out = {}
    for name in names:
        per_gpu = NET_BATCH[name]
        global_batch = per_gpu * world
        net, (lo, hi) = nets.build_shard(name, global_batch, rank, world)
        dn = nets.device_net(net, device)
        dn.input.normal_()
        dn.capture()
        for _ in range(3):
            dn.replay()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(dn.stream):  # graph replays go to the current stream
            e0.record(dn.stream)
            for _ in range(steps):
                dn.graph.replay()
            e1.record(dn.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ms], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        sec = ms / 1e3
        line = {
            "samples_per_s": round(global_batch * steps / sec, 1),
            "tflops": round(net.flops * world * steps / sec / 1e12, 2),
            "ms_per_forward": round(ms / steps, 4),
            "batch_per_gpu": per_gpu, "global_batch": global_batch,
            "launches_per_forward": dn.launches,
            "sharding": f"batch across {world} GPU(s), no collective" if world > 1 else "single GPU",
            "dtype": "fp16 activations / fp32 accumulate",
            "weights": "random init (no checkpoints offline)",
        }
        if isinstance(net, nets.BertDef):
            line.update(seq=net.seq, layers=net.layers, tokens_per_s=round(global_batch * net.seq * steps / sec, 1),
                        graph="encoder stack (embedding lookup excluded)")
        else:
            line.update(image=net.input_shape[1], images_per_s=line["samples_per_s"])
        out[name] = line
        del dn
        torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------- CPU reference

def cpu_reference_sample(name, budget_s, threads):
    """tir::run (reference interpreter, oracle/_ref) on `threads` disjoint output
    slices of the workload, concurrently. Returns (TFLOPS, seconds, sample text)."""
    from oracle import ir_gen as G
    from oracle import oracle as O

    spec = op_spec(name)
    ospec = G.ConvSpec(op=spec.op, n=spec.n, in_dhw=spec.in_dhw, ci=spec.ci, co=spec.co, k=spec.k,
                       s=spec.s, p=spec.p, d=spec.d, groups=spec.groups,
                       transposed=spec.transposed)
    od, oh, ow = ospec.out_dhw()
    macs_per_pixel = ospec.macs() // (ospec.n * od * oh * ow)
    ns_per_mac = 1.3e-6  # survey-measured tir::run cost on conv
    pix = max(1, int(budget_s / (macs_per_pixel * ns_per_mac)))
    pix = min(pix, ow)
    X = O.reference_tensor(ospec.x_shape(), 1)
    W = O.reference_tensor(ospec.w_shape(), 2)
    rows_total = ospec.n * od * oh
    texts = []
    for t in range(threads):
        r = (t * 7919) % rows_total
        texts.append(G.conv_source(ospec, rows=(r, r + 1), cols=(0, pix)))
    wall = O.ref_run_many(texts, [X, W])
    macs = threads * pix * macs_per_pixel
    return 2 * macs / wall / 1e12, wall, (
        f"{threads} concurrent tir::run slices of {name} image rows, {pix} output pixels x "
        f"{macs_per_pixel} MACs each ({macs} MACs total)")


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O

    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtirref.so not built"}))
        return
    threads = os.cpu_count() or 1
    total_budget = 150.0
    per_step = max(0.5, total_budget / (args.steps + args.warmup))
    for _ in range(args.warmup):
        cpu_reference_sample(HEADLINE, per_step, threads)
    vals, secs = [], 0.0
    sample = ""
    for _ in range(args.steps):
        v, s, sample = cpu_reference_sample(HEADLINE, per_step, threads)
        vals.append(v)
        secs += s
    value = statistics.mean(vals)
    spec = op_spec(HEADLINE)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference distribution, workloads.h:170-184)",
        "config": {"workload": f"{HEADLINE} N{spec.n} {spec.in_dhw[1]}x{spec.in_dhw[2]}x{spec.ci}->"
                               f"{spec.co} 3x3 s1 p1 (bounded per-step sample)",
                   "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": "TFLOPS", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ----------------------------------------------------------------------------- main

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--op", default=HEADLINE)
    ap.add_argument("--no-ops", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-nets", action="store_true", help="skip the batch-sharded network forwards")
    ap.add_argument("--nets", default="resnet50,mobilenet_v2,bert_large")
    ap.add_argument("--profile", metavar="OP", help="eager launches of one op for ncu (no timing)")
    ap.add_argument("--profile-range", metavar="OP",
                    help="a CUDA graph of --steps launches of one op, replayed between cudaProfilerStart/Stop "
                         "(ncu --graph-profiling graph: steady-state DRAM bytes and time per launch)")
    ap.add_argument("--launcher-check", action="store_true",
                    help="rank bookkeeping only (gloo, no GPU): one JSON line with the ranks seen")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world, rank, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        spawn_ranks(args.gpus)
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        sys.exit(2)
    if args.launcher_check:
        import torch

        dist = init_dist(world, "gloo")
        seen = torch.tensor([rank], dtype=torch.int64)
        if dist:
            got = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(got, seen)
            ranks = sorted(int(t.item()) for t in got)
            dist.destroy_process_group()
        else:
            ranks = [rank]
        if rank == 0:
            print(json.dumps({"n_gpus": world, "ranks": ranks}), flush=True)
        return

    if args.profile_range:
        import torch

        # the K launches are captured into one CUDA graph (tensor maps are encoded at
        # capture), and only its replay lies between cudaProfilerStart / Stop:
        # `ncu --graph-profiling graph --profile-from-start off` then reports the
        # whole graph as one result (DRAM bytes incl. write-backs, total time)
        r = OpRunner(args.profile_range, torch.device("cuda", 0))
        for i in range(args.warmup):
            r.step(i)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        steps = max(args.steps, r.sets)  # every rotating set once: the graph's data exceeds 2x L2
        with torch.cuda.graph(g, capture_error_mode="relaxed"):
            for i in range(steps):
                r.step(args.warmup + i)
        print(json.dumps({"profile_range": args.profile_range, "launches": steps, "sets": r.sets}), flush=True)
        g.replay()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
        g.replay()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
        return

    if args.profile:
        import torch

        r = OpRunner(args.profile, torch.device("cuda", 0))
        for i in range(args.warmup + args.steps):
            r.step(i)
        torch.cuda.synchronize()
        return

    if args.impl == "reference":
        run_reference(args)
        return

    import torch

    torch.cuda.set_device(local)
    dist = init_dist(world, "nccl")
    device = torch.device("cuda", local)
    pk = peaks()

    name = args.op
    runner = OpRunner(name, device)
    ms, launches, clocks = time_graph(runner, args.steps, args.warmup, dist,
                                      sampler_gpu=local if rank == 0 else None)
    flops, byts, bound = op_work(name)
    sec = ms / 1e3
    value = flops * args.steps * world / sec / 1e12
    kernel_s = sec / args.steps  # one launch per step
    if bound == "hbm":
        achieved, peak, unit = byts / kernel_s / 1e9, pk["hbm_gbs"], "GB/s"
    else:
        achieved, peak, unit = flops / kernel_s / 1e12, pk["bf16_tflops"], "TFLOP/s"
    n_sets = runner.sets
    del runner
    torch.cuda.empty_cache()

    floor_us = None
    ops = {}
    if not args.no_ops and rank == 0:
        try:  # per-launch floor: a one-CTA GEMM in the same graph-replay regime
            r = OpRunner("FLOOR", device)
            fms, _, _ = time_graph(r, 100, 3, None, None)
            floor_us = fms / 100 * 1e3
            del r
        except Exception as e:
            floor_us = None
            ops["FLOOR"] = {"error": str(e)[:200]}
        for other in SWEEP:
            try:
                r = OpRunner(other, device)
                k = max(10, min(args.steps, 100)) if other != "GMM8K" else 10
                oms, ol, _ = time_graph(r, k, 3, None, None)
                f, b, bd = op_work(other)
                t = oms / 1e3 / k
                t_roof = max(f / (pk["bf16_tflops"] * 1e12), b / (pk["hbm_gbs"] * 1e9))
                ops[other] = {
                    "tflops": round(f / t / 1e12, 2), "gbs": round(b / t / 1e9, 1),
                    "us": round(t * 1e6, 3), "bound": bd,
                    "frac_tensor_spec": round(f / t / 1e12 / SPEC_TC_PEAK_TFLOPS, 4),
                    "frac_tensor_measured": round(f / t / 1e12 / pk["bf16_tflops"], 4),
                    "frac_hbm": round(b / t / 1e9 / pk["hbm_gbs"], 4),
                    # roofline time / measured time (not clamped)
                    "frac_roofline": round(t_roof / t, 4),
                    # the same with the measured per-launch floor taken out of the measured time
                    "frac_roofline_ex_floor": (round(t_roof / max(t - floor_us * 1e-6, t_roof), 4)
                                               if floor_us else None),
                    "roofline_us": round(t_roof * 1e6, 3),
                    "launches_per_step": ol / k, "l2_sets": r.sets,
                    "algorithmic_bytes": b, "algorithmic_flops": f,
                    "traffic_per_launch": traffic_from_profiles(other),
                }
                del r
                torch.cuda.empty_cache()
            except Exception as e:  # report, never hide
                ops[other] = {"error": str(e)[:200]}

    net_lines = {}
    if not args.no_nets:
        try:
            net_lines = measure_nets(device, world, rank, dist, max(5, min(args.steps, 20)),
                                     [n for n in args.nets.split(",") if n])
        except Exception as e:  # report, never hide
            net_lines = {"error": str(e)[:300]}

    e2e = None
    e2e_interp = None
    if not args.no_e2e and rank == 0:
        e2e = measure_e2e(name, args.steps)
        try:
            e2e_interp = measure_e2e_interp(name)
        except Exception as e:  # report, never hide
            e2e_interp = {"error": str(e)[:300]}

    cpu = None
    if not args.no_cpu and rank == 0:
        try:
            threads = os.cpu_count() or 1
            v, s, sample = cpu_reference_sample(name, 10.0, threads)
            cpu = {"value": v, "unit": "TFLOPS", "cores": threads, "kind": "reference",
                   "sample": sample, "seconds": round(s, 2)}
        except Exception as e:
            cpu = {"value": None, "unit": "TFLOPS", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"[:200]}

    if rank == 0:
        spec = op_spec(name)
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "TFLOPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 6),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16",
            "data": "synthetic N(0,1)->fp16 inputs created on device",
            "config": {
                "workload": (f"{name} N{spec.n} {spec.in_dhw[1]}x{spec.in_dhw[2]}x{spec.ci}->{spec.co} "
                             f"{spec.k[1]}x{spec.k[2]} s{spec.s[2]} p{spec.p[2]}, fp16 in / fp32 acc / fp32 out"
                             if spec else "GMM 1024^3"),
                "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                "l2": f"rotating {n_sets} input/output sets > 2x L2 (126 MB)",
                "timing": "CUDA graph of K launches, CUDA events on the launching stream",
            },
            "frac_of_spec_tensor_peak": round(value / world / SPEC_TC_PEAK_TFLOPS, 4),
            "roofline": {"bound": bound, "achieved": round(achieved, 2), "peak": peak, "unit": unit,
                         "frac": round(achieved / peak, 4), "traffic": traffic_from_profiles(name),
                         "algorithmic_bytes": byts, "algorithmic_flops": flops,
                         "peak_source": pk["source"]},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks,
            "gpu_launches": launches,
            "launches_per_step": launches / args.steps,
            "floor_us": round(floor_us, 3) if floor_us else None,
            "e2e_interp": e2e_interp,
            "ops": ops,
            "nets": net_lines,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
