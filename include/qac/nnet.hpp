// qac/nnet.hpp -- drop-in replacement for the reference header of the same
// name (/root/reference/proj/include/qac/nnet.hpp:1-104).  Put this
// repository's include/ directory BEFORE the reference's include/ on the
// compiler's include path: every `#include "qac/nnet.hpp"` in the reference
// (pipeline.hpp:18, reference.hpp:7, cli.hpp:10, bindings/qac_module.cpp:13)
// then resolves here, and qac::nnet::* is the B200 implementation
// (qac_b200.hpp, libga3c_b200.so).
#pragma once

#include "qac/returns.hpp"
#include "../qac_b200.hpp"

namespace qac {
namespace nnet = ::qac_b200::nnet;
}  // namespace qac
