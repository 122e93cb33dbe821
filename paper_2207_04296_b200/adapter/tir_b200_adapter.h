// tir_b200_adapter.h — the reference-side plugin: registers B200 intrinsics as
// HostKernels on the UNCHANGED reference API (/root/reference/proj/include/tir/interp.h).
//
//   using HostKernel = std::function<void(std::vector<TensorView>&)>;   // interp.h:120
//   ExecContext::register_host_kernel(name, kernel)                      // interp.h:125
//
// A block annotated "tensorized" whose body is `b200.gmm()` (or a conv
// intrinsic name registered here) is dispatched by Interp::dispatch_call
// (src/interp.cc:360-383) with views [writes[0], reads...] in signature order;
// the kernel accumulates into the output window, exactly like the reference's
// own intrinsic test kernel (tests/test_interp.cc:180-193). No `exec_scope`
// annotation may be put on these whole-op blocks (TH-SCOPE, validate.cc:432-455).
//
// Error behaviour mirrors the reference: tir::Error(kind, msg) (ir.h:33-48)
// with kinds ValueError (bad views, inexact fp16 input), UnsupportedShape and
// CudaError. Duplicate registration raises DuplicateName (interp.cc:149).
#ifndef TIR_B200_ADAPTER_H_
#define TIR_B200_ADAPTER_H_

#include <string>

#include "tir/interp.h"
#include "tir_b200.h"

namespace tir_b200 {

// GMM intrinsic: views [C f32 [M,N], A f16 [M,K], B f16 [K,N]]; C += A.B
// (accumulate = true, the blockize convention), or C = A.B (accumulate = false:
// the whole-op composite folded a zero init into the call, so C is neither
// read nor uploaded).
void register_gmm(tir::ExecContext& ctx, const std::string& name = "b200.gmm", bool accumulate = true);

// Convolution intrinsic with fixed geometry (the reference forwards neither
// call arguments nor annotations to the kernel, interp.cc:360-383, so stride,
// padding, dilation and groups are captured here). Views [Y, X, W] whose
// extents must match the descriptor (tir_b200.h layouts).
void register_conv(tir::ExecContext& ctx, const std::string& name, const tir_b200_conv_desc& desc,
                   bool accumulate = true);

// The conventional intrinsic name for a descriptor, e.g. "b200.c2d.s1p1d1g1".
std::string conv_intrin_name(const tir_b200_conv_desc& desc);

}  // namespace tir_b200

#endif  // TIR_B200_ADAPTER_H_
