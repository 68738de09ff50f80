#pragma once
#include <exception>
#include <string>

#include "util.h"

namespace tpx {

extern thread_local std::string g_last_error;

// Run `f`, converting any exception into TPX_ERR + g_last_error (never throw across the ABI).
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 1;
  } catch (...) {
    g_last_error = "unknown error";
    return 1;
  }
}

}  // namespace tpx

#define TPX_API extern "C" __attribute__((visibility("default")))
