#pragma once
// hp_status -> the reference's exception types: the C++ face of
// the C-ABI keeps the reference's error contract -- std::invalid_argument
// for bad input (proj/src/*: fail()), hetplan::infeasible_error
// (types.hpp:15-17), std::runtime_error otherwise (CUDA/NCCL/timeouts).

#include <stdexcept>
#include <string>

#include "hetplan/types.hpp"
#include "hp_capi.h"

namespace hetplan {

inline void check(hp_status s) {
    if (s == HP_OK) return;
    const std::string msg = hp_last_error();
    switch (s) {
        case HP_EINVAL: throw std::invalid_argument(msg);
        case HP_EINFEASIBLE: throw infeasible_error(msg);
        default: throw std::runtime_error(msg);
    }
}

}  // namespace hetplan
