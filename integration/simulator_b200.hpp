// Reference-side adapter over the B200 executor's C ABI (see simulator_b200.cpp).
#pragma once
#include <cstdint>
#include <string>

#include "tileplan/simulator.hpp"

namespace tileplan {

// execute_numeric (proj/include/tileplan/simulator.hpp:43) on cuda:0 through libtpx.so.
// precision: TPX_PREC_TF32 / TPX_PREC_FP32; flags: TPX_FLAG_* (include/tpx.h).
NumericCheck execute_numeric_b200(const ExecutionPlan& p, std::uint64_t seed, int precision, int flags);
// tpx_plan_describe of the plan lowered host-only for `rank` of `world` (JSON).
std::string describe_b200(const ExecutionPlan& p, int rank, int world, int flags);

}  // namespace tileplan
