// tir_b200_tensorize.h — caller-side whole-op tensorize composite.
//
// Lets an unchanged scalar workload PrimFunc route to the B200 kernels through
// the reference's own schedule API:
//
//   1. match_contraction recognises the block as GMM or one of the paper's
//      convolutions (C1D/C2D/C3D/DIL/GRP/T2D/DEP). The recognition is the
//      paper's characteristic-vector test (SPEC.md "characteristic_vectors" /
//      "propose_mapping"): every iterator's (Y, X, W) membership, plus the affine
//      form of the input index for stride, dilation and padding
//      (linear_terms, include/tir/analysis.h).
//   2. tensorize_whole_op blockizes the block's outermost loop
//      (Schedule::blockize, src/schedule_block.cc:407-610; init moves to the
//      outer block). It requires an extent-1 outer block, i.e. the loop nest
//      covers the whole op. Then it replaces the outer block's body with
//      `<intrin>()` + attrs("tensorized" = <intrin>) and records the step
//      "b200.tensorize" through Schedule::commit_rewrite (schedule.cc:348-352).
//   3. register_tensorize_step_handler makes that step replayable from a trace
//      (register_step_handler, schedule.cc:354-363 / apply_step :760-766).
//
// The generated intrinsic name encodes the full geometry, so one ExecContext
// can carry several convs. register_matched binds it to the B200 kernel
// (tir_b200_adapter.h).
//
// Errors are tir::Error kinds: DescMismatch (not a recognised contraction),
// NotSeparable / StaleHandle (from blockize), NotWholeOp (a sliced nest).
#ifndef TIR_B200_TENSORIZE_H_
#define TIR_B200_TENSORIZE_H_

#include <string>

#include "tir/interp.h"
#include "tir/schedule.h"
#include "tir/text.h"
#include "tir_b200.h"

namespace tir_b200 {

struct OpMatch {
  bool gmm = false;
  int64_t m = 0, n = 0, k = 0;  // GMM extents
  tir_b200_conv_desc conv{};    // conv geometry (when !gmm)
  std::string intrin;           // generated intrinsic name
  bool overwrite = false;       // the block's zero init was folded into the call (Y = op, suffix ".ow")
};

// Recognises `block` in f (see above). Throws DescMismatch with the reason.
OpMatch match_contraction(const tir::PrimFunc& f, const std::string& block);

// The composite primitive. Returns the match; the tensorized block is the
// outer block blockize created (its name is in the recorded trace step).
OpMatch tensorize_whole_op(tir::Schedule& s, const std::string& block);

// Registers the B200 HostKernel for a match on ctx (no-op if the name is taken).
void register_matched(tir::ExecContext& ctx, const OpMatch& m);

// Registers the replay handler for "b200.tensorize" trace steps (idempotent).
void register_tensorize_step_handler();

// the channel pad of small-CI convolutions (CI = 3 stems) as
// reference schedule steps instead of a device relayout. On a conv block in the
// direct form (one loop per iterator, per-element read regions):
//   cache_read(block, 0), cache_read(block, 1)   -- stage X and W (schedule_block.cc:283)
//   pad_block(block, rc -> padded)               -- grow the reduction to `padded`
//                                                   channels, zero-filling the staged
//                                                   copies (schedule_block.cc:1186)
//   b200.widen_reads(block)                      -- declare whole-buffer read regions
//                                                   (a conservative over-approximation)
//                                                   so a later whole-op tensorize sees
//                                                   in-bounds operand windows
// Every step is recorded in the trace; the last one replays through
// register_step_handler (registered here). Returns the padded reduction extent.
int64_t pad_conv_channels(tir::Schedule& s, const std::string& block, int64_t multiple);

// Full-geometry intrinsic name, e.g. "b200.c2d.n16_i1x56x56_c64_o64_k1x3x3_s1x1x1_p0x1x1_d1x1x1_g1".
std::string conv_intrin_key(const tir_b200_conv_desc& d);

// Intrinsic declarations in the reference grammar (`intrin NAME { require P
// scope("global") contiguous ... }`, parser.cc:749-781, text.h:45-59).
// intrin_decl_text emits the declaration of a matched intrinsic: its operands
// (views [writes[0], reads...], named after the block's buffers) must be
// global, row-major, innermost-contiguous — what the C-ABI consumes — and, as
// whole-op blocks must, it carries no exec_scope (TH-SCOPE, validate.cc:432-455).
// register_declared builds the B200 HostKernel registry from a parsed program
// alone: the full geometry is in the intrinsic name (conv_intrin_key, plus
// ".ow" for the overwriting form), so each `b200.*` declaration is decoded and
// registered; a declaration asking for anything else (another scope, an
// exec_scope, an undecodable name) throws DescMismatch. Returns the count.
std::string intrin_decl_text(const OpMatch& m, const std::vector<std::string>& operands);
int register_declared(tir::ExecContext& ctx, const tir::ParsedProgram& program);
// Decodes an intrinsic name produced by tensorize_whole_op (inverse of conv_intrin_key).
OpMatch decode_intrin(const std::string& name);

}  // namespace tir_b200

#endif  // TIR_B200_TENSORIZE_H_
