// Kernel instantiations: target __nv_bfloat16, drafts float.
#define COSINE_TT __nv_bfloat16
#define COSINE_TQ float
#define COSINE_SET kernel_set_bf
#include "k_dtype.inc"
