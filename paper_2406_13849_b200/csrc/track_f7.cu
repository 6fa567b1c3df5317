// Kernels for models with any surface kind and hex arrays.
#define NT_FEAT 15
#define NT_NS f7
#include "track_impl.cuh"
