// C ABI plumbing: per-thread last-error text and the ABI version.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace tidas {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

}  // namespace tidas

extern "C" const char* tidas_last_error(void) { return tidas::g_err; }

extern "C" int tidas_abi_version(void) { return 6; }  // 2: tidas_das_desc_t.window, tidas_das_window; 3: .geometry; 4: tidas_das_image_peers;
// 5: tidas_rf_analytic_range, tidas_das_window_range; 6: tidas_rf_analytic_ex (TIDAS_K1_RF_READY)
