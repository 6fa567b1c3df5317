// The rect-specialised tracker under the ring scheduler (k_track_event with RTK != 0): its own
// translation unit, so that its instantiations compile in parallel with the generic ones.
#define NT_FEAT 0
#define NT_NS f0r
#define NT_RECT_TU 1
#include "track_impl.cuh"
