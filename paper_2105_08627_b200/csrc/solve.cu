// Saddle-system operator (Eq. 7) and preconditioned GMRES solve.
#include "internal.h"

namespace svh {
void free_solve(svh_handle*) {}
}  // namespace svh

using namespace svh;
extern "C" {
int svh_apply_system(svh_handle*, const void*, void*, int32_t, svh_stream) {
    set_error("svh_apply_system: not implemented yet");
    return SVH_EINVAL;
}
int svh_solve(svh_handle*, const svh_port*, int32_t, double*, double*, double*, double*, svh_stats*) {
    set_error("svh_solve: not implemented yet");
    return SVH_EINVAL;
}
int svh_solve_columns(svh_handle*, const svh_port*, int32_t, const int32_t*, int32_t, double*, svh_stats*) {
    set_error("svh_solve_columns: not implemented yet");
    return SVH_EINVAL;
}
}
