// layout.hpp -- flat parameter layout of the extended NetworkSpec.
//
// Reproduces nnet.cpp:29-45 (Slice/Layout/layout_of) for FC layers and the
// heads, and prepends VALID NHWC conv layers stored OHWI (W[Cout][k][k][Cin]
// then b[Cout]).  For a conv layer the weight row of output channel co is the
// K-major GEMM operand B[co][(ky,kx,ci)], so the implicit-GEMM kernels read
// the parameter vector directly without repacking.
#pragma once

#include <cstddef>
#include <cstdint>

#include "ga3c.h"

namespace ga3c {

struct Layer {
  bool is_conv = false;
  int cin = 0, cout = 0, k = 0, stride = 0;  // conv geometry
  int ih = 0, iw = 0, oh = 0, ow = 0;
  int in = 0, out = 0;  // GEMM fan-in (k*k*cin for conv) and fan-out
  std::size_t w_off = 0, b_off = 0;
  int out_dim() const { return is_conv ? oh * ow * cout : out; }
  int in_dim() const { return is_conv ? ih * iw * cin : in; }
  int pixels() const { return is_conv ? oh * ow : 1; }
};

struct Layout {
  Layer trunk[GA3C_MAX_CONV + GA3C_MAX_HIDDEN];
  int n_trunk = 0;
  int n_conv = 0;
  Layer policy, value;
  std::size_t total = 0;
  int in_dim = 0;
  int n_actions = 0;
  int head_in() const { return policy.in; }
  int max_act_dim() const {
    int m = in_dim;
    for (int i = 0; i < n_trunk; ++i)
      if (trunk[i].out_dim() > m) m = trunk[i].out_dim();
    return m;
  }
};

int validate_spec(const ga3c_net_spec& s);
int validate_hyper(const ga3c_hyper& hp);
Layout layout_of(const ga3c_net_spec& s);

// splitmix64 / mt19937_64 / next_uniform (util.hpp:19-43), used by the host
// init so the device starts from exactly the reference's draws.
std::uint64_t mix64(std::uint64_t x);
void init_params(const Layout& lo, std::uint64_t seed, double* theta64);

}  // namespace ga3c
