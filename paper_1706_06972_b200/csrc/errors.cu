// Error channel of the C-ABI: last message per host thread.
#include <atomic>
#include <string>

#include "common.cuh"

namespace ocsc {
static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(OCSC_ECUDA, std::string(cudaGetErrorName(e)) + " (" + cudaGetErrorString(e) + ") in " + where);
}
}  // namespace ocsc

extern "C" const char* ocsc_last_error(void) { return ocsc::g_last_error.c_str(); }
extern "C" int ocsc_abi_version(void) { return OCSC_ABI_VERSION; }
extern "C" int64_t ocsc_kernel_launches(void) { return ocsc::g_launches.load(); }
