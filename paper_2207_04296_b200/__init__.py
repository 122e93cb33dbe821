"""paper_2207_04296_b200 — B200-native (sm_100a) tensorized operator set of
arXiv 2207.04296 (TensorIR): GMM, C1D, C2D, C3D, DIL, GRP, T2D on tcgen05
tensor cores and DEP on CUDA cores, behind the C-ABI of include/tir_b200.h and
the reference's HostKernel API (adapter/)."""
from .api import (  # noqa: F401
    GMM_SHAPE,
    PAPER_SHAPES,
    Conv,
    TirError,
    compulsory_bytes,
    avgpool_global,
    layernorm,
    maxpool2d,
    softmax,
    conv,
    conv_host,
    gmm,
    gmm_batched,
    gmm_host,
    launch_count,
    lib,
    reset_launch_count,
    set_option,
    get_option,
    useful_macs,
)
