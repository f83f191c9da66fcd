// tcgen05/TMEM sgemm emitter (placeholder until the kernel lands).
#include <string>

#include "ispc.h"
#include "nest_view.hpp"

namespace ispc {

std::string emit_tcgen05_kernel(const ispc_tile_config& c, const std::string& fn, ispc_launch& L) {
  (void)c;
  (void)fn;
  (void)L;
  throw NestError(ISPC_E_ILLEGAL, "tcgen05 sgemm not available in this build");
}

}  // namespace ispc
