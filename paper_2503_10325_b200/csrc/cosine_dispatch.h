// cosine_dispatch.h — the kernel set of one (target dtype, draft dtype, draft kind, N) combination.
//
// The heavy kernel templates are instantiated once per dtype pair in their own translation
// unit (k_<tt><tq>.cu, compiled in parallel); the host code (cosine_abi.cu) picks a set here.
#pragma once

#include "cosine_tree.cuh"

namespace cosine {

using SplitFn = void (*)(SplitParams);
using TreeFn = void (*)(TreeParams);

struct KernelSet {
  SplitFn stats;         // stats_kernel (lazy rounds, tree all-nodes, sharded)
  SplitFn lazy_decide;   // lazy round decisions (NEXT-1)
  SplitFn decide;        // split path decisions (stats -> decide -> resample)
  SplitFn sample_decide; // the same with SAMPLE selection (x* ~ fused q)
  SplitFn stats_slices;  // SAMPLE over probability drafts: stats_kernel + 64-group slice sums
  SplitFn sample_decide_w;  // ... and its warp-per-unit draw from the slices (nullptr: logits)
  SplitFn fuse_decide;   // cosine_fuse_drafts: Eq. 4 fusion per unit
  SplitFn fuse_write_q;  // cosine_fuse_drafts: the fused distribution rows
  SplitFn sample_prep;   // cosine_sample_residual: the request records
  SplitFn resample;      // final draws
  SplitFn tiny;          // small batches: the three steps in one cooperative launch
  SplitFn shard_pack;    // vocabulary-sharded records
  SplitFn shard_sample;  // vocabulary-sharded owner scan
  TreeFn tree_decide;
  TreeFn tree_walk;
};

void kernel_set_bb(bool logits, int N, KernelSet* out);  // bf16 target, bf16 drafts
void kernel_set_bf(bool logits, int N, KernelSet* out);  // bf16 target, fp32 drafts
void kernel_set_fb(bool logits, int N, KernelSet* out);  // fp32 target, bf16 drafts
void kernel_set_ff(bool logits, int N, KernelSet* out);  // fp32 target, fp32 drafts

}  // namespace cosine
