// Housekeeping entry points of the C ABI: version, thread-local last error,
// launch counter (evidence that the native path ran; see bench.py).
#include <string>

#include "ab_common.cuh"

namespace ab {
std::atomic<int64_t> g_launches{0};
static thread_local std::string t_err;
void set_error(const std::string& msg) { t_err = msg; }
}  // namespace ab

extern "C" {
int ab_version(void) { return 100; }  // 0.1.0
const char* ab_last_error(void) { return ab::t_err.c_str(); }
int64_t ab_launch_count(void) { return ab::g_launches.load(); }

}
