// Kernels for models with rect arrays, CSG cells of axis planes and z-cylinders only.
#define NT_FEAT 0
#define NT_NS f0
#include "track_impl.cuh"
