// Rect-specialised tracker tables (filled in by a later milestone).
#include "nt_model.hpp"

namespace nt {
void build_rect_tables(const std::vector<HSurf>&, const std::vector<HMat>&, const std::vector<HCell>&,
                       const std::vector<HUniv>&, int, Flat& F) {
  F.rect_ok = false;
  F.rect_why = "rect tracker not built yet";
}
}  // namespace nt
