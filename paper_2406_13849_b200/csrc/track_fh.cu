// The default path (SP ring kernel, no trace or tallies) for models with hex arrays and general
// planes but no spheres or non-uniform rect arrays: a smaller kernel than f7's (instruction fetch).
#define NT_FEAT 3
#define NT_NS fh
#define NT_EVENT_TU 1
#include "track_impl.cuh"
