// qac/returns.hpp -- drop-in replacement for the reference header of the
// same name (/root/reference/proj/include/qac/returns.hpp:1-32): the
// Experience / ExperienceBatch types and compute_returns of qac_b200.hpp
// (n-step returns on the device, fp64, bitwise) under the reference's names.
#pragma once

#include "../qac_b200.hpp"

namespace qac {
namespace returns = ::qac_b200::returns;
}  // namespace qac
