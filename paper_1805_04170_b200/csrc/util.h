#pragma once
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

namespace tpx {

// Mirrors tileplan::Error (proj/include/tileplan/error.hpp:8-12): every failure is an
// exception inside the library; the C ABI turns it into a status code + tpx_last_error().
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

[[noreturn]] inline void fail(const std::string& msg) { throw Error(msg); }

}  // namespace tpx

#define CUDA_CHECK(expr)                                                                  \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      throw ::tpx::Error(std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " + \
                         __FILE__ + ":" + std::to_string(__LINE__) + " (" #expr ")");     \
  } while (0)
