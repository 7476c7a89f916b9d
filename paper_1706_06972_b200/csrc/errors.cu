// Error channel of the C-ABI: last message per host thread.
#include <string>

#include "common.cuh"

namespace ocsc {
static thread_local std::string g_last_error;

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
