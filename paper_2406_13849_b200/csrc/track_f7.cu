// Kernels for models with any surface kind and hex arrays.
#ifndef NT_F7_FEAT
#define NT_F7_FEAT 15
#endif
#define NT_FEAT NT_F7_FEAT
#define NT_NS f7
#include "track_impl.cuh"
