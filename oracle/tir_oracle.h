/*
 * tir_oracle.h — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * Plain-C restatement of the reference interpreter's semantics for the tensorized
 * operator set, used only by tests/ and bench.py's cpu_baseline leg as a checker.
 * Pinned against the reference itself: tests/test_oracle.py runs the same
 * programs through tir::run (oracle/_ref/libtirref.so, built from
 * /root/reference/proj/src) and through the committed golden vectors in
 * tests/golden/, and requires value equality.
 *
 * Semantics followed (file:line under /root/reference/proj):
 *   - every float op is an fp32 op; mul and add are separate rounded ops
 *     (src/interp.cc:484-512; compiled with -ffp-contract=off);
 *   - the reduction starts from init = 0.0 (or from the prior output value when
 *     accumulating, tests/test_interp.cc:186) and runs in loop order:
 *     k innermost for GMM (tests/testing/workloads.h:42-44), (rd, rh, rw, rc)
 *     for conv (workloads.h:106-108), (rh, rw) for depthwise (workloads.h:146-147);
 *   - padded taps contribute select(inb, x, 0.0) * w, i.e. acc + 0*w
 *     (the `select` form used by oracle/ir_gen.py, src/interp.cc:463-466);
 *   - F16 operands are f32 values (include/tir/ir.h:52-53, src/interp.cc:67-78).
 */
#ifndef TIR_ORACLE_H_
#define TIR_ORACLE_H_

#include <stdint.h>

#include "../include/tir_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* C[M,N] = (acc ? C : 0) + A[M,K] . B[K,N], k-sequential fp32. */
int tir_oracle_gmm(const float* A, const float* B, float* C, int64_t M, int64_t N, int64_t K,
                   int accumulate, int threads);

/* Y = (acc ? Y : 0) + conv(X, W) for every op of tir_b200_conv_desc (C1D..DEP). */
int tir_oracle_conv(const tir_b200_conv_desc* d, const float* X, const float* W, float* Y,
                    int accumulate, int threads);

/* Output extents, same formula as the product (tir_b200.h). */
int tir_oracle_conv_out(const tir_b200_conv_desc* d, int64_t out[3]);

#ifdef __cplusplus
}
#endif

#endif
