"""GPU tests of the network graphs: ResNet-50 and
MobileNet-V2 forwards through the C-ABI (every conv / GEMM on the tcgen05
kernels with fused bias / residual / ReLU(6), DEP on the CUDA-core kernel, the
pooling glue) against the float64 CPU replay of the same op list
(oracle/nets_ref.py), which rounds activations to fp16 exactly where the device
graph does. Tolerance: the device reassociates fp32 sums inside the tensor
cores, which flips an fp16 rounding now and then; those 1-ulp (2^-11) flips
propagate but stay far below 2% of the logit range.

Also: the glue kernels alone (exact: max is exact, mean / LayerNorm / softmax
to fp32 rounding), the fused residual epilogue on both conv paths, CUDA-graph
replay == eager, and batch-shard consistency (two half-batch graphs == one
full-batch graph)."""
import numpy as np
import pytest
import torch

import paper_2207_04296_b200 as tb
from paper_2207_04296_b200 import nets

pytestmark = pytest.mark.gpu

LOGIT_TOL = 2e-2


def _rel(got, want):
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-6))


@pytest.mark.parametrize("name", ["resnet50", "mobilenet_v2"])
def test_network_matches_cpu_reference(name, cuda):
    from oracle import nets_ref

    net = nets.NETS[name](2, image=64)
    dn = nets.DeviceNet(net, cuda)
    x = np.random.default_rng(1).standard_normal(net.input_shape).astype(np.float16)
    dn.input.copy_(torch.from_numpy(x))
    with torch.cuda.stream(dn.stream):
        dn.run()
    dn.stream.synchronize()
    got = dn.output.reshape(2, -1).cpu().numpy()
    want = nets_ref.forward(net, x)
    assert np.isfinite(got).all()
    assert _rel(got, want) < LOGIT_TOL, _rel(got, want)
    assert (got.argmax(1) == want.argmax(1)).all()


@pytest.mark.parametrize("name", ["resnet50", "mobilenet_v2"])
def test_graph_replay_equals_eager_and_shards(name, cuda):
    net = nets.NETS[name](4, image=64)
    dn = nets.DeviceNet(net, cuda)
    x = torch.randn(net.input_shape, device=cuda).half()
    dn.input.copy_(x)
    with torch.cuda.stream(dn.stream):
        dn.run()
    dn.stream.synchronize()
    eager = dn.output.clone()
    dn.capture()
    dn.output.zero_()
    dn.replay()
    torch.cuda.synchronize()
    assert torch.equal(dn.output, eager)
    # two ranks' shards (same seed = replicated weights), evaluated independently
    parts = []
    for r in range(2):
        sub, (lo, hi) = nets.build_shard(name, 4, r, 2, image=64)
        ds = nets.DeviceNet(sub, cuda)
        ds.input.copy_(x[lo:hi])
        with torch.cuda.stream(ds.stream):
            ds.run()
        ds.stream.synchronize()
        parts.append(ds.output)
    full = torch.cat(parts)
    assert _rel(full.cpu().numpy(), eager.cpu().numpy()) < 1e-2


def test_maxpool_avgpool_exact(cuda):
    g = torch.Generator(device=cuda).manual_seed(3)
    x = torch.randn(3, 17, 15, 24, device=cuda, generator=g).half()
    y = tb.maxpool2d(x, 3, 2, 1)
    want = torch.nn.functional.max_pool2d(x.float().permute(0, 3, 1, 2), 3, 2, 1).permute(0, 2, 3, 1)
    assert torch.equal(y.float(), want)
    a = tb.avgpool_global(x)
    wa = x.double().mean(dim=(1, 2)).half()
    assert (a.float() - wa.float()).abs().max().item() <= 1e-3 * wa.float().abs().max().item()


def test_layernorm_softmax(cuda):
    g = torch.Generator(device=cuda).manual_seed(4)
    x = torch.randn(37, 1024, device=cuda, generator=g).half()
    gamma = torch.randn(1024, device=cuda, generator=g)
    beta = torch.randn(1024, device=cuda, generator=g)
    y = tb.layernorm(x, gamma, beta, 1e-12)
    want = torch.nn.functional.layer_norm(x.double(), (1024,), gamma.double(), beta.double(), 1e-12)
    assert (y.double() - want).abs().max().item() < 2e-2
    s = tb.softmax(x, 0.125)
    ws = torch.softmax(x.double() * 0.125, dim=-1)
    assert (s.double() - ws).abs().max().item() < 1e-3


@pytest.mark.parametrize("shape", [
    dict(op="C2D", n=2, in_dhw=(1, 14, 14), ci=64, co=64, k=(1, 3, 3), p=(0, 1, 1)),        # halo path
    dict(op="C2D", n=2, in_dhw=(1, 15, 15), ci=64, co=128, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1)),  # im2col
])
@pytest.mark.parametrize("act", ["relu", "relu6", "none"])
def test_conv_residual_epilogue(shape, act, cuda):
    from oracle import oracle as O

    spec = tb.Conv(**shape)
    X = O.reference_tensor(spec.x_shape(), 1)
    W = O.reference_tensor(spec.w_shape(), 2)
    R = O.reference_tensor(spec.y_shape(), 3)
    bias = O.reference_tensor((spec.co,), 4)
    got = tb.conv(spec, torch.from_numpy(X).to(cuda).half(), torch.from_numpy(W).to(cuda).half(),
                  bias=torch.from_numpy(bias).to(cuda), relu=act,
                  residual=torch.from_numpy(R).to(cuda).half()).cpu().numpy()
    v = O.conv(O.ConvSpec(**shape), X, W, threads=8) + bias + R  # exact on the reference distribution
    if act == "relu":
        v = np.maximum(v, 0)
    elif act == "relu6":
        v = np.clip(v, 0, 6)
    assert O.tensors_bitwise_equal(got, v.astype(np.float32))


def test_gmm_residual_gelu(cuda):
    g = torch.Generator(device=cuda).manual_seed(5)
    a = torch.randn(256, 128, device=cuda, generator=g).half()
    b = torch.randn(128, 96, device=cuda, generator=g).half()
    r = torch.randn(256, 96, device=cuda, generator=g).half()
    bias = torch.randn(96, device=cuda, generator=g)
    y = tb.gmm(a, b, out_f16=True, bias=bias, residual=r, relu="gelu")
    want = torch.nn.functional.gelu(a.double() @ b.double() + bias.double() + r.double())
    assert (y.double() - want).abs().max().item() < 2e-2
    with pytest.raises(tb.TirError):
        tb.gmm(a, b, relu="swish")


@pytest.mark.parametrize("n_dim", [64, 256])
def test_gmm_batched_strided_heads(n_dim, cuda):
    """Per-(sequence, head) problems over strided views, as in attention."""
    g = torch.Generator(device=cuda).manual_seed(6)
    B, nh, S, dh = 2, 3, 128, 64
    qkv = torch.randn(B * S, 3 * nh * dh, device=cuda, generator=g).half()
    kt = torch.randn(nh * dh, B * S, device=cuda, generator=g).half()
    out = torch.zeros(B * nh * S, S, device=cuda).half()
    tb.gmm_batched(qkv, kt, out, S, S, dh, (B, nh), a=((0, S, 0), (0, 0, dh)), b=((0, 0, dh), (0, S, 0)),
                   c=((0, nh * S, S), (0, 0, 0)))
    for b in range(B):
        for h in range(nh):
            want = qkv[b * S:(b + 1) * S, h * dh:(h + 1) * dh].double() @ kt[h * dh:(h + 1) * dh, b * S:(b + 1) * S].double()
            got = out[(b * nh + h) * S:(b * nh + h + 1) * S].double()
            assert (got - want).abs().max().item() <= 2e-3 * want.abs().max().item() + 1e-2
    # P V: N = dh (64) or a wider slice
    p = torch.randn(B * nh * S, S, device=cuda, generator=g).half()
    v = torch.randn(B * S, nh * n_dim, device=cuda, generator=g).half()
    ctx = torch.zeros(B * S, nh * n_dim, device=cuda).half()
    tb.gmm_batched(p, v, ctx, S, n_dim, S, (B, nh), a=((0, nh * S, S), (0, 0, 0)), b=((0, S, 0), (0, 0, n_dim)),
                   c=((0, S, 0), (0, 0, n_dim)))
    for b in range(B):
        for h in range(nh):
            want = p[(b * nh + h) * S:(b * nh + h + 1) * S].double() @ v[b * S:(b + 1) * S, h * n_dim:(h + 1) * n_dim].double()
            got = ctx[b * S:(b + 1) * S, h * n_dim:(h + 1) * n_dim].double()
            assert (got - want).abs().max().item() <= 2e-3 * want.abs().max().item() + 1e-2


def test_gmm_batched_kmajor_b(cuda):
    """B given as [N, K] (K contiguous): attention's K read in place from QKV."""
    g = torch.Generator(device=cuda).manual_seed(8)
    B, nh, S, dh = 2, 3, 128, 64
    H = nh * dh
    qkv = torch.randn(B * S, 3 * H, device=cuda, generator=g).half()
    out = torch.zeros(B * nh * S, S, device=cuda).half()
    tb.gmm_batched(qkv, qkv, out, S, S, dh, (B, nh), a=((0, S, 0), (0, 0, dh)), b=((0, S, 0), (H, 0, dh)),
                   c=((0, nh * S, S), (0, 0, 0)), b_kmajor=True)
    for b in range(B):
        for h in range(nh):
            q = qkv[b * S:(b + 1) * S, h * dh:(h + 1) * dh].double()
            k = qkv[b * S:(b + 1) * S, H + h * dh:H + (h + 1) * dh].double()
            want = q @ k.t()
            got = out[(b * nh + h) * S:(b * nh + h + 1) * S].double()
            assert (got - want).abs().max().item() <= 2e-3 * want.abs().max().item() + 1e-2
    # wider K (two 64-deep sub-blocks) and N = 256 tiles
    a = torch.randn(2 * 256, 128, device=cuda, generator=g).half()
    bt = torch.randn(2 * 256, 128, device=cuda, generator=g).half()
    c = torch.zeros(2 * 256, 256, device=cuda).half()
    tb.gmm_batched(a, bt, c, 256, 256, 128, (2, 1), a=((0, 256, 0), (0, 0, 0)), b=((0, 256, 0), (0, 0, 0)),
                   c=((0, 256, 0), (0, 0, 0)), b_kmajor=True)
    for z in range(2):
        want = a[z * 256:(z + 1) * 256].double() @ bt[z * 256:(z + 1) * 256].double().t()
        assert (c[z * 256:(z + 1) * 256].double() - want).abs().max().item() <= 2e-3 * want.abs().max().item() + 1e-2


def test_gmm_batched_rejects_bad_windows(cuda):
    a = torch.zeros(128, 64, device=cuda).half()
    c = torch.zeros(128, 64, device=cuda).half()
    with pytest.raises(tb.TirError):
        tb.gmm_batched(a, a, c, 128, 64, 64, (2, 1), a=((0, 128, 0), (0, 0, 0)), b=((0, 0, 0), (0, 0, 0)),
                       c=((0, 0, 0), (0, 0, 0)))


def test_bert_matches_cpu_reference(cuda):
    from oracle import nets_ref

    net = nets.bert_large(2, seq=128, layers=2, hidden=128, heads=2, ffn=512)
    dn = nets.device_net(net, cuda)
    x = np.random.default_rng(2).standard_normal(net.input_shape).astype(np.float16)
    dn.input.copy_(torch.from_numpy(x))
    with torch.cuda.stream(dn.stream):
        dn.run()
    dn.stream.synchronize()
    got = dn.output.float().cpu().numpy()
    want = nets_ref.bert_forward(net, x)
    err = np.abs(got - want)
    assert np.isfinite(got).all()
    assert err.max() < 5e-2 and err.mean() < 2e-3, (err.max(), err.mean())
    # CUDA graph replay reproduces the eager forward exactly
    dn.input.copy_(torch.from_numpy(x))
    dn.capture()  # warm-up run inside capture() overwrites the input in place (x -> layer output)
    dn.input.copy_(torch.from_numpy(x))
    dn.replay()
    torch.cuda.synchronize()
    assert np.array_equal(dn.output.float().cpu().numpy(), got)


CUDA_SHARD_WORKER = """
import os, sys
sys.path.insert(0, {root!r})
import numpy as np, torch, torch.distributed as dist
from paper_2207_04296_b200 import nets
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)  # one GPU on the test box: both ranks share it
dev = torch.device("cuda", 0)
outs = {{}}
for name, B, kw in (("resnet50", 4, dict(image=64)), ("mobilenet_v2", 4, dict(image=64)),
                    ("bert_large", 2, dict(seq=128, layers=2, hidden=128, heads=2, ffn=512))):
    if name == "bert_large":
        from paper_2207_04296_b200 import shard
        lo, hi = shard.batch_range(B, rank, world)
        net = nets.bert_large(hi - lo, **kw)
    else:
        net, (lo, hi) = nets.build_shard(name, B, rank, world, **kw)
    full_shape = (B,) + tuple(net.input_shape[1:]) if name != "bert_large" else (B * kw["seq"], kw["hidden"])
    x = np.random.default_rng(5).standard_normal(full_shape).astype(np.float16)
    xs = x[lo:hi] if name != "bert_large" else x[lo * kw["seq"]:hi * kw["seq"]]
    dn = nets.device_net(net, dev)
    dn.input.copy_(torch.from_numpy(xs))
    dn.capture()                      # the warm-up run inside capture() consumed the input
    dn.input.copy_(torch.from_numpy(xs))
    dn.replay()
    torch.cuda.synchronize()
    part = dn.output.float().cpu().numpy()
    parts = [None] * world
    dist.all_gather_object(parts, part)
    if rank == 0:
        if name == "bert_large":
            fnet = nets.bert_large(B, **kw)
        else:
            fnet = nets.NETS[name](B, **kw)
        fd = nets.device_net(fnet, dev)
        fd.input.copy_(torch.from_numpy(x))
        with torch.cuda.stream(fd.stream):
            fd.run()
        fd.stream.synchronize()
        full = fd.output.float().cpu().numpy()
        got = np.concatenate(parts)
        outs[name] = bool(got.shape == full.shape and np.array_equal(got, full))
if rank == 0:
    print("CUDA_SHARDS", outs, flush=True)
    print("CUDA_SHARD_OK" if outs and all(outs.values()) else "CUDA_SHARD_BAD", flush=True)
dist.destroy_process_group()
"""


def test_two_rank_cuda_shards_bitwise_equal_full_batch(tmp_path):
    """two ranks (gloo for the gather; the test box has one GPU, so
    both run on cuda:0) each run their batch shard of ResNet-50 / MobileNet-V2 /
    a small BERT through libtir_b200 as a captured CUDA graph; the gathered
    output equals the one-process full-batch forward BIT FOR BIT (no collective
    in the hot path; fused-epilogue layers keep one reduction order per element
    whatever the batch)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "cuda_shard_worker.py"
    script.write_text(CUDA_SHARD_WORKER.format(root=root))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29561", str(script)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert "CUDA_SHARD_OK" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]


@pytest.mark.parametrize("name", ["resnet50", "mobilenet_v2"])
def test_network_full_size_matches_cpu_reference(name, cuda):
    """The benchmarked configuration (224 x 224 images, every layer at full
    width) against the float64 CPU replay, B = 2; and two graph replays give
    bit-identical logits."""
    from oracle import nets_ref

    net = nets.NETS[name](2, image=224)
    dn = nets.DeviceNet(net, cuda)
    x = np.random.default_rng(11).standard_normal(net.input_shape).astype(np.float16)
    dn.input.copy_(torch.from_numpy(x))
    dn.capture()
    dn.input.copy_(torch.from_numpy(x))
    dn.replay()
    torch.cuda.synchronize()
    got = dn.output.reshape(2, -1).cpu().numpy().copy()
    dn.replay()
    torch.cuda.synchronize()
    assert np.array_equal(dn.output.reshape(2, -1).cpu().numpy(), got)
    want = nets_ref.forward(net, x)
    rel = _rel(got, want)
    print(f"[full-size] {name}: max |logit err| / max |logit| = {rel:.3e}")
    assert np.isfinite(got).all()
    assert rel < LOGIT_TOL, rel
    assert (got.argmax(1) == want.argmax(1)).all()


def test_bert_large_full_size_matches_cpu_reference(cuda):
    """BERT-large at the benchmarked dimensions (hidden 1024, 16 heads, FFN 4096,
    24 layers, sequence 512, B = 1) against the float64 CPU replay with the
    device graph's fp16 rounding points."""
    from oracle import nets_ref

    net = nets.bert_large(1, seq=512)
    assert (net.hidden, net.heads, net.layers, net.seq) == (1024, 16, 24, 512)
    dn = nets.device_net(net, cuda)
    x = np.random.default_rng(12).standard_normal(net.input_shape).astype(np.float16)
    dn.input.copy_(torch.from_numpy(x))
    with torch.cuda.stream(dn.stream):
        dn.run()
    dn.stream.synchronize()
    got = dn.output.float().cpu().numpy()
    want = nets_ref.bert_forward(net, x)
    err = np.abs(got - want)
    cos = float(np.sum(got * want) / np.sqrt(np.sum(got * got) * np.sum(want * want)))
    print(f"[full-size] bert_large: max err {err.max():.3e}, mean err {err.mean():.3e}, cosine {cos:.8f}")
    assert np.isfinite(got).all()
    assert cos > 0.9999 and err.mean() < 1e-2, (err.max(), err.mean(), cos)
