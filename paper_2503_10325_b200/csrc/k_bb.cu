// Kernel instantiations: target __nv_bfloat16, drafts __nv_bfloat16.
#define COSINE_TT __nv_bfloat16
#define COSINE_TQ __nv_bfloat16
#define COSINE_SET kernel_set_bb
#include "k_dtype.inc"
