"""GPU diagnostic sweep (not collected by pytest): runs every operator case in
its own subprocess (a trapped kernel cannot poison the next case) and prints
one line per case: parity vs the oracle (bit-exact on the reference
distribution) and a rough device time.

    python tests/gpu_diag.py            # all cases
    python tests/gpu_diag.py CASE       # one case, in-process
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CASES = {
    "gmm_1tile": ("gmm", (128, 64, 64)),
    "gmm_256x128x256": ("gmm", (256, 128, 256)),
    "gmm_odd_m": ("gmm", (200, 64, 128)),
    "gmm_k72": ("gmm", (128, 64, 72)),
    "gmm_n48": ("gmm", (256, 48, 128)),
    "gmm_1024": ("gmm", (1024, 1024, 1024)),
    "gmm_2048x512x768": ("gmm", (2048, 512, 768)),
    "c2d_small": ("conv", dict(op="C2D", n=2, in_dhw=(1, 8, 8), ci=64, co=64, k=(1, 3, 3), p=(0, 1, 1))),
    "c2d_nopad": ("conv", dict(op="C2D", n=1, in_dhw=(1, 10, 12), ci=64, co=128, k=(1, 3, 3))),
    "c2d_s2": ("conv", dict(op="C2D", n=2, in_dhw=(1, 15, 15), ci=128, co=64, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1))),
    "c2d_ci32": ("conv", dict(op="C2D", n=2, in_dhw=(1, 9, 9), ci=32, co=64, k=(1, 3, 3), p=(0, 1, 1))),
    "c2d_ci16": ("conv", dict(op="C2D", n=2, in_dhw=(1, 9, 9), ci=16, co=32, k=(1, 3, 3), p=(0, 1, 1))),
    "c2d_ci8": ("conv", dict(op="C2D", n=2, in_dhw=(1, 9, 9), ci=8, co=16, k=(1, 3, 3), p=(0, 1, 1))),
    "c2d_paper": ("conv", "C2D"),
    "c1d_paper": ("conv", "C1D"),
    "grp_small": ("conv", dict(op="GRP", n=2, in_dhw=(1, 12, 12), ci=64, co=128, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1), groups=4)),
    "grp_paper": ("conv", "GRP"),
    "dil_small": ("conv", dict(op="DIL", n=1, in_dhw=(1, 30, 30), ci=3, co=64, k=(1, 7, 7), s=(1, 2, 2), p=(0, 3, 3), d=(1, 2, 2))),
    "c3d_small": ("conv", dict(op="C3D", n=1, in_dhw=(6, 12, 12), ci=3, co=64, k=(7, 7, 7), s=(2, 2, 2), p=(3, 3, 3))),
    "t2d_small": ("conv", dict(op="T2D", n=2, in_dhw=(1, 4, 4), ci=64, co=64, k=(1, 4, 4), s=(1, 2, 2), p=(0, 1, 1), transposed=True)),
    "t2d_paper": ("conv", "T2D"),
    "dep_small": ("conv", dict(op="DEP", n=2, in_dhw=(1, 9, 9), ci=32, co=32, k=(1, 3, 3), p=(0, 1, 1), groups=32)),
    "dep_paper": ("conv", "DEP"),
    "dep_s2": ("conv", dict(op="DEP", n=2, in_dhw=(1, 28, 28), ci=96, co=96, k=(1, 3, 3), s=(1, 2, 2), p=(0, 1, 1), groups=96)),
    "dil_paper": ("conv", "DIL"),
    "halo_c2d_ci128": ("conv", dict(op="C2D", n=2, in_dhw=(1, 14, 14), ci=128, co=128, k=(1, 3, 3), p=(0, 1, 1))),
    "halo_c2d_wide": ("conv", dict(op="C2D", n=1, in_dhw=(1, 6, 150), ci=64, co=64, k=(1, 3, 3), p=(0, 1, 1))),
    "halo_c2d_dil2": ("conv", dict(op="C2D", n=2, in_dhw=(1, 20, 20), ci=64, co=32, k=(1, 3, 3), p=(0, 2, 2), d=(1, 2, 2))),
    "halo_c2d_5x5_nopad": ("conv", dict(op="C2D", n=2, in_dhw=(1, 17, 19), ci=64, co=96, k=(1, 5, 5))),
    "halo_grp_s1": ("conv", dict(op="GRP", n=2, in_dhw=(1, 12, 12), ci=128, co=128, k=(1, 3, 3), p=(0, 1, 1), groups=2)),
    "halo_c2d_co256": ("conv", dict(op="C2D", n=1, in_dhw=(1, 28, 28), ci=64, co=256, k=(1, 3, 3), p=(0, 1, 1))),
}


def run_case(name):
    import torch

    import paper_2207_04296_b200 as tb
    from oracle import oracle as O

    kind, arg = CASES[name]
    dev = torch.device("cuda:0")
    res = {"case": name}
    if kind == "gmm":
        M, N, K = arg
        A = O.reference_tensor((M, K), 1)
        B = O.reference_tensor((K, N), 2)
        Ad = torch.from_numpy(A).to(dev).half()
        Bd = torch.from_numpy(B).to(dev).half()
        C = tb.gmm(Ad, Bd)
        torch.cuda.synchronize()
        got = C.cpu().numpy()
        rows = min(M, 256)
        ref = O.gmm(A[:rows], B, threads=8)
        res["exact"] = bool(O.tensors_bitwise_equal(got[:rows], ref))
        res["maxdiff"] = float(np.abs(got[:rows] - ref).max())
        # accumulate + fp16 out variants
        C2 = torch.from_numpy(O.reference_tensor((M, N), 3)).to(dev)
        C2h = C2.cpu().numpy()
        tb.gmm(Ad, Bd, C2, accumulate=True)
        Ch = tb.gmm(Ad, Bd, out_f16=True)
        torch.cuda.synchronize()
        res["acc_exact"] = bool(O.tensors_bitwise_equal(C2.cpu().numpy()[:rows], O.gmm(A[:rows], B, C2h[:rows], threads=8)))
        res["f16_exact"] = bool(np.array_equal(Ch.cpu().numpy()[:rows], ref.astype(np.float16)))
        flops = 2 * M * N * K
        fn = lambda: tb.gmm(Ad, Bd, C)  # noqa: E731
    else:
        if isinstance(arg, str):
            spec = tb.PAPER_SHAPES[arg]
        else:
            spec = tb.Conv(**arg)
        X = O.reference_tensor(spec.x_shape(), 1)
        W = O.reference_tensor(spec.w_shape(), 2)
        Xd = torch.from_numpy(X).to(dev).half()
        Wd = torch.from_numpy(W).to(dev).half()
        Y = tb.conv(spec, Xd, Wd)
        torch.cuda.synchronize()
        got = Y.cpu().numpy()
        from oracle.ir_gen import ConvSpec
        ospec = ConvSpec(op=spec.op, n=spec.n, in_dhw=spec.in_dhw, ci=spec.ci, co=spec.co, k=spec.k,
                         s=spec.s, p=spec.p, d=spec.d, groups=spec.groups, transposed=spec.transposed)
        # check the first image (outputs are independent per image)
        ospec1 = ConvSpec(**{**ospec.__dict__, "n": 1})
        ref = O.conv(ospec1, X[:1], W, threads=8)
        res["exact"] = bool(O.tensors_bitwise_equal(got[:1], ref))
        res["maxdiff"] = float(np.abs(got[:1] - ref).max())
        bad = np.argwhere(got[:1] != ref)
        res["nbad"] = int(len(bad))
        if len(bad):
            res["first_bad"] = [int(v) for v in bad[0]]
        if spec.n > 1:
            ospecl = ConvSpec(**{**ospec.__dict__, "n": 1})
            refl = O.conv(ospecl, X[-1:], W, threads=8)
            res["exact_last"] = bool(O.tensors_bitwise_equal(got[-1:], refl))
        flops = 2 * tb.useful_macs(spec)
        fn = lambda: tb.conv(spec, Xd, Wd, Y)  # noqa: E731
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    n = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    res["us"] = round(ms * 1e3, 2)
    res["tflops"] = round(flops / (ms * 1e-3) / 1e12, 1)
    print(json.dumps(res), flush=True)


def main():
    if len(sys.argv) > 1 and sys.argv[1] != "--all":
        for c in sys.argv[1:]:
            run_case(c)
        return
    for name in CASES:
        t0 = time.time()
        try:
            p = subprocess.run([sys.executable, __file__, name], capture_output=True, text=True, timeout=120)
            out = p.stdout.strip().splitlines()
            line = out[-1] if out else ""
            if p.returncode != 0 or not line.startswith("{"):
                err = (p.stderr.strip().splitlines() or ["?"])[-1]
                print(json.dumps({"case": name, "error": err[-300:], "rc": p.returncode}), flush=True)
            else:
                print(line, flush=True)
        except subprocess.TimeoutExpired:
            print(json.dumps({"case": name, "error": "timeout"}), flush=True)
        sys.stderr.write(f"{name}: {time.time() - t0:.1f}s\n")


if __name__ == "__main__":
    main()
