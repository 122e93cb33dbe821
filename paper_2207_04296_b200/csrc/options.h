// options.h — planner switches of libtir_b200 (host side).
//
// The defaults are the measured best (DESIGN.md §5 "Switches"); every switch
// only changes HOW an operator is planned (tile shape, pipeline depth, epilogue
// flavour), never its result, and every variant is parity-tested. They are
// read ONCE, at the first planner call, from TIR_B200_<NAME> environment
// variables, and can be changed afterwards through tir_b200_set_option() —
// nothing is re-read per launch.
#pragma once

#include <cstdlib>
#include <cstring>
#include <mutex>

namespace tb {

struct Options {
  // value -1 = automatic (planner decides)
  int no_pdl = 0;          // 1: no programmatic dependent launch
  int mc = 1;              // 0: no tcgen05.mma.cta_group::2 GEMM pairs
  int max_ctas = 0;        // > 0: cap the persistent grid
  int epi8 = -1;           // 0 / 1: force the 4- or 8-warp igemm epilogue
  int ks = 0;              // > 0: K sub-blocks per igemm stage
  int ks_strict = 0;       // 1: narrow-piece convs keep the two-stage shared-memory limit
  int no_tma_store = 0;    // 1: generic register-store epilogues only
  int bn = 0;              // > 0: force the igemm N tile
  int ksplit = 0;          // > 0: force the split-K factor (cluster-reduced, deterministic)
  int no_halo = 0;         // 1: stride-1 convs take the im2col kernel
  int igemm_prefetch = 0;  // 1: im2col producers prefetch the first stage's A into L2 before the PDL wait
  int no_gpack = 0;        // 1: grouped convs with 16 / 32 channels per group take one narrow im2col piece per group
  int no_rowpack = 0;      // 1: CI = 3 stems / C3D take the (kw, c) relayout + im2col kernel
  int rp_backoff = 64;     // rowpack: ns between barrier polls of producers / epilogue (0: spin)
  int rp_backoff2 = 0;     // rowpack: same for the builders
  int rowpack_debug = 0;   // timing experiments only, WRONG results: 1 no raw loads in the builders, 2 no stores
  int pack_hw = -1;        // 0 / 1: disable / force the (kh, kw, c) relayout of CI % 8 != 0 layers
  int pack_kw = 1;         // 0: no (kw, c) relayout
  int pack_gather = 0;     // 1: gather form of the (kw, c) relayout for dilated strips
  int dep_simple = 0;      // 1: DEP takes the untiled kernel
  int dep_tc = 0;          // 8 / 16: DEP stride-1 tile-width override
  int no_smem_bias = 0;    // 1: never stage the bias in shared memory
  int host_chunks = 8;     // host-buffer calls: batch chunks of the H2D / conv / D2H pipeline
  int host_pipeline = 1;   // 0: host-buffer calls do not pipeline batch chunks
  int l2_prefetch = 2;     // 0: the halo conv does not prefetch its first tile into L2 before the PDL
                           // wait; 1: it also prefetches the whole weight panel (2: one box per CTA) (measured: the same prefetch in igemm / DEP cost 0.7-1.7 us — the
                           // prefetches occupy the TMA queue ahead of the real loads — so only halo has it)
};

struct OptionEntry {
  const char* name;
  using Field = int Options::*;
  Field field;
};

inline const OptionEntry* option_table(int* count) {
  static const OptionEntry t[] = {
      {"no_pdl", &Options::no_pdl},         {"mc", &Options::mc},
      {"max_ctas", &Options::max_ctas},     {"epi8", &Options::epi8},
      {"ks", &Options::ks},                 {"ks_strict", &Options::ks_strict},
      {"no_tma_store", &Options::no_tma_store}, {"bn", &Options::bn},
      {"ksplit", &Options::ksplit},         {"no_halo", &Options::no_halo},
      {"no_rowpack", &Options::no_rowpack},     {"no_gpack", &Options::no_gpack},
      {"igemm_prefetch", &Options::igemm_prefetch},     {"rowpack_debug", &Options::rowpack_debug},
      {"rp_backoff", &Options::rp_backoff},     {"rp_backoff2", &Options::rp_backoff2},
      {"pack_hw", &Options::pack_hw},       {"pack_kw", &Options::pack_kw},
      {"pack_gather", &Options::pack_gather}, {"dep_simple", &Options::dep_simple},
      {"dep_tc", &Options::dep_tc},         {"no_smem_bias", &Options::no_smem_bias},
      {"host_pipeline", &Options::host_pipeline},
      {"host_chunks", &Options::host_chunks}, {"l2_prefetch", &Options::l2_prefetch},
  };
  *count = static_cast<int>(sizeof t / sizeof t[0]);
  return t;
}

// Process-wide switches, initialised from the environment on first use.
inline Options& options() {
  static Options o;
  static std::once_flag once;
  std::call_once(once, [] {
    int n = 0;
    const OptionEntry* t = option_table(&n);
    for (int i = 0; i < n; ++i) {
      char var[64] = "TIR_B200_";
      for (int j = 0; t[i].name[j] && j < 50; ++j) {
        const char c = t[i].name[j];
        var[9 + j] = (c >= 'a' && c <= 'z') ? static_cast<char>(c - 32) : c;
        var[10 + j] = 0;
      }
      if (const char* e = getenv(var)) o.*(t[i].field) = atoi(e);
    }
  });
  return o;
}

}  // namespace tb
