"""CPU tests of the host side: the C-ABI library loads and exports every entry
point include/tir_b200.h declares (no compute without a GPU), descriptor
validation runs on the host, the product does not link the oracle, and the
batch-sharding logic holds across a 2-rank gloo group."""
import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from paper_2207_04296_b200 import api, shard

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tir_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void|const char\*)\s+(tir_b200_\w+)\s*\(",
                                 text, flags=re.M)))


def test_header_declares_the_boundary():
    fns = declared_functions()
    for f in ["tir_b200_gmm", "tir_b200_conv", "tir_b200_gmm_host", "tir_b200_conv_host",
              "tir_b200_gmm_host_f32", "tir_b200_conv_host_f32", "tir_b200_last_error",
              "tir_b200_conv_out_shape"]:
        assert f in fns


def test_library_exports_every_declared_symbol():
    lib = api.lib()
    for f in declared_functions():
        assert hasattr(lib, f), f


def test_product_does_not_link_the_oracle():
    out = subprocess.run(["ldd", api.LIB_PATH], capture_output=True, text=True).stdout
    assert "tirkit" not in out and "tir_oracle" not in out and "tirref" not in out
    syms = subprocess.run(["nm", "-D", api.LIB_PATH], capture_output=True, text=True).stdout
    assert "tir_oracle" not in syms and "tirref" not in syms


def test_product_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "-lelf", api.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", api.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass          # tcgen05.mma
    assert "UTMALDG" in sass          # TMA loads
    assert "IM2COL" in sass           # im2col TMA (implicit GEMM)
    assert "LDTM" in sass             # tcgen05.ld (TMEM -> registers)
    assert "HMMA" not in re.sub(r"UTCHMMA", "", sass)  # no legacy mma.sync path


@pytest.mark.parametrize("op", list(api.PAPER_SHAPES))
def test_out_shape_on_host(op):
    spec = api.PAPER_SHAPES[op]
    from oracle.ir_gen import PAPER_SHAPES as OS

    assert spec.out_dhw() == OS[op].out_dhw()


def test_descriptor_validation_errors():
    bad = api.Conv("C2D", n=1, in_dhw=(1, 2, 2), ci=4, co=4, k=(1, 5, 5))
    with pytest.raises(api.TirError) as e:
        bad.out_dhw()
    assert e.value.kind == "ValueError"
    with pytest.raises(api.TirError) as e:
        api.Conv("GRP", n=1, in_dhw=(1, 4, 4), ci=6, co=4, k=(1, 3, 3), groups=4).out_dhw()
    assert e.value.kind == "ValueError"
    with pytest.raises(api.TirError):
        api.Conv("C2D", n=0, in_dhw=(1, 4, 4), ci=4, co=4, k=(1, 1, 1)).out_dhw()


def test_error_string_is_thread_local_and_set():
    lib = api.lib()
    d = api.Conv("C2D", n=1, in_dhw=(1, 2, 2), ci=4, co=4, k=(1, 5, 5)).desc()
    out = (ctypes.c_int64 * 3)()
    assert lib.tir_b200_conv_out_shape(ctypes.byref(d), out) == api.ERR_VALUE
    assert b"kernel" in lib.tir_b200_last_error()


def test_paper_shape_bookkeeping():
    c2d = api.PAPER_SHAPES["C2D"]
    assert api.useful_macs(c2d) * 2 == 3699376128
    assert api.compulsory_bytes(c2d) == 19341312


@pytest.mark.parametrize("batch,world", [(16, 2), (16, 3), (5, 8), (1, 1)])
def test_batch_ranges_partition(batch, world):
    seen = []
    for r in range(world):
        lo, hi = shard.batch_range(batch, r, world)
        seen.extend(range(lo, hi))
    assert seen == list(range(batch))


WORKER = r"""
import os, sys
sys.path.insert(0, {root!r})
import numpy as np, torch, torch.distributed as dist
from oracle import oracle as O, ir_gen as G
from paper_2207_04296_b200 import shard
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
spec = G.ConvSpec("C2D", n=5, in_dhw=(1, 6, 6), ci=8, co=8, k=(1, 3, 3), p=(0, 1, 1))
x = O.reference_tensor(spec.x_shape(), 1); w = O.reference_tensor(spec.w_shape(), 2)
sub, (lo, hi) = shard.shard_spec(spec, rank, world)
y = O.conv(sub, x[lo:hi], w) if hi > lo else np.zeros((0,) + spec.y_shape()[1:], np.float32)
parts = [None] * world
dist.all_gather_object(parts, y)
t = shard.max_over_ranks(float(rank + 1), dist)
if rank == 0:
    full = O.conv(spec, x, w)
    ok = O.tensors_bitwise_equal(np.concatenate(parts), full) and t == world
    print("SHARD_OK" if ok else "SHARD_BAD", flush=True)
dist.destroy_process_group()
"""


def test_two_rank_gloo_batch_shard(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(WORKER.format(root=ROOT))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", str(script)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
    assert "SHARD_OK" in p.stdout, p.stdout + p.stderr


def test_bench_reference_arm_help():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True,
                       text=True, timeout=120)
    assert p.returncode == 0 and "--impl" in p.stdout


def test_host_api_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    A = np.zeros((128, 64), np.float16)
    B = np.zeros((64, 64), np.float16)
    with pytest.raises(api.TirError) as e:
        api.gmm_host(A, B)
    assert e.value.kind == "CudaError"


def test_bench_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` outside torchrun re-executes itself under
    torch.distributed.run with two ranks (gloo bookkeeping only, no GPU)."""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launcher-check"],
                       capture_output=True, text=True, timeout=300)
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert p.returncode == 0 and lines, p.stdout + p.stderr
    import json

    d = json.loads(lines[-1])
    assert d == {"n_gpus": 2, "ranks": [0, 1]}
    # a WORLD_SIZE that contradicts --gpus is an error, not a silent 1-GPU run
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launcher-check"],
                       capture_output=True, text=True, timeout=120, env=env)
    assert p.returncode == 2 and "WORLD_SIZE" in p.stdout
