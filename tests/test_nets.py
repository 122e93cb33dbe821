"""CPU tests of the network graphs: graph structure and
work counts, and the batch-sharded runner logic across a 2-rank gloo group (each
rank evaluates its shard with the CPU reference; the gathered shards must equal
the full-batch result)."""
import os
import subprocess
import sys

import numpy as np

from paper_2207_04296_b200 import nets

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_resnet50_structure_and_flops():
    net = nets.resnet50(1)
    kinds = [op.kind for op in net.ops]
    # 53 convolutions (1 stem + 16 bottlenecks x 3 + 4 projections) + FC
    assert kinds.count("conv") + kinds.count("gmm") == 54
    assert kinds.count("maxpool") == 1 and kinds.count("avgpool") == 1
    assert net.shapes[net.output] == (1, 1, 1, 1000)
    # ~4.1 G multiply-adds per 224x224 image
    assert abs(net.flops / 2 / 4.1e9 - 1) < 0.03, net.flops
    assert sum(1 for op in net.ops if op.res) == 16
    assert nets.launches_per_forward(net) == len(net.ops) + 2  # CI=3 stem relayout


def test_mobilenet_v2_structure_and_flops():
    net = nets.mobilenet_v2(1)
    assert sum(1 for op in net.ops if op.kind == "dep") == 17
    assert sum(1 for op in net.ops if op.res) == 10
    assert abs(net.flops / 2 / 300e6 - 1) < 0.05, net.flops
    assert net.shapes[net.output] == (1, 1, 1, 1000)


def test_shards_replicate_weights():
    a, (lo, hi) = nets.build_shard("resnet50", 5, 1, 2, image=32)
    b = nets.resnet50(5, image=32)
    assert (lo, hi) == (3, 5) and a.batch == 2
    for x, y in zip(a.ops, b.ops):
        assert x.kind == y.kind
        if x.w is not None:
            assert np.array_equal(x.w, y.w) and np.array_equal(x.b, y.b)


def test_reference_forward_small():
    from oracle import nets_ref

    net = nets.mobilenet_v2(2, image=32)
    x = np.random.default_rng(0).standard_normal(net.input_shape).astype(np.float16)
    y = nets_ref.forward(net, x)
    assert y.shape == (2, 1000) and np.isfinite(y).all() and np.abs(y).max() > 0


WORKER = """
import os, sys
sys.path.insert(0, {root!r})
import numpy as np, torch.distributed as dist
from paper_2207_04296_b200 import nets, shard
from oracle import nets_ref
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
B = 3
net, (lo, hi) = nets.build_shard("resnet50", B, rank, world, image=32)
x = np.random.default_rng(7).standard_normal((B, 32, 32, 3)).astype(np.float16)
y = nets_ref.forward(net, x[lo:hi])
parts = [None] * world
dist.all_gather_object(parts, y)
if rank == 0:
    full = nets_ref.forward(nets.resnet50(B, image=32), x)
    got = np.concatenate(parts)
    ok = got.shape == full.shape and np.allclose(got, full, rtol=1e-9, atol=1e-9)
    print("NET_SHARD_OK" if ok else "NET_SHARD_BAD", float(np.abs(got - full).max()), flush=True)
dist.destroy_process_group()
"""


def test_two_rank_gloo_network_shard(tmp_path):
    script = tmp_path / "net_worker.py"
    script.write_text(WORKER.format(root=ROOT))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29541")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", str(script)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
    assert "NET_SHARD_OK" in p.stdout, p.stdout + p.stderr


def test_bert_structure_and_flops():
    net = nets.bert_large(1, seq=512)
    assert net.layers == 24 and net.hidden == 1024 and net.heads == 16 and net.head_dim == 64
    # ~335 M parameters in the encoder stack's GEMMs (24 x 12.6 M)
    params = sum(v.size for w in net.weights for k, v in w.items() if k.startswith("w_"))
    assert abs(params / 24 / 12.58e6 - 1) < 0.01
    # per 512-token sequence: dense 2 x 512 x 12.58M x 24 + attention 4 x 16 x 512^2 x 64 x 24
    assert net.flops == 24 * (2 * 512 * (4 * 1024 * 1024 + 2 * 1024 * 4096) + 4 * 16 * 512 * 512 * 64)
    assert nets.launches_per_forward(net) == 216


def test_bert_reference_small():
    from oracle import nets_ref

    net = nets.bert_large(2, seq=128, layers=2, hidden=128, heads=2, ffn=512)
    x = np.random.default_rng(0).standard_normal(net.input_shape).astype(np.float16)
    y = nets_ref.bert_forward(net, x)
    assert y.shape == net.input_shape and np.isfinite(y).all()
    # post-LN output: every token row normalised (then scaled by ~1 gamma)
    assert np.abs(y.mean(axis=1)).max() < 0.5
