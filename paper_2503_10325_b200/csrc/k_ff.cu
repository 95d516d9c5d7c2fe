// Kernel instantiations: target float, drafts float.
#define COSINE_TT float
#define COSINE_TQ float
#define COSINE_SET kernel_set_ff
#include "k_dtype.inc"
