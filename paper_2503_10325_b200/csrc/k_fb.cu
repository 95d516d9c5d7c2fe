// Kernel instantiations: target float, drafts __nv_bfloat16.
#define COSINE_TT float
#define COSINE_TQ __nv_bfloat16
#define COSINE_SET kernel_set_fb
#include "k_dtype.inc"
