// qac_b200.hpp -- the reference's value-type math API on the B200 device.
//
// Same names, argument meaning and error behaviour as the reference
// `qac::nnet` (include/qac/nnet.hpp:14-104) and `qac::returns`
// (include/qac/returns.hpp:13-32), implemented over the C ABI
// (include/ga3c.h).  A caller written against the reference --
// predictor_loop, trainer_main, SharedModel::apply, train_sync, the pybind
// module -- switches with an include path: include/qac/nnet.hpp and
// include/qac/returns.hpp shadow the reference headers of the same names and
// alias qac::nnet / qac::returns to the namespaces below, so the reference's
// own sources compile unmodified against this library (INTEGRATION.md §2,
// oracle/Makefile target `dropin`).
//
// Semantics kept:
//   * pure value semantics: every call takes theta by const& and returns new
//     vectors; nothing is cached across calls, so in-place edits of theta
//     (finite-difference tests) are always seen;
//   * std::invalid_argument for the reference's validation failures
//     (nnet.cpp:75-81,123-145,178-179,206-228; returns.cpp:10-17);
//   * rmsprop_update returns applied=false with inputs unchanged for a
//     non-finite gradient (nnet.cpp:299-301);
//   * concurrent calls from different threads are safe (each thread owns its
//     device contexts).
// Differences, by design: the device computes in fp32 (3xTF32 GEMMs), so
// doubles are rounded to fp32 on the way in; results match the fp64
// reference within the tolerances in DESIGN.md §2.  Returns are bitwise.
//
// Extension: NetworkSpec carries optional conv layers; the
// reference's {input_dim, hidden_dims, n_actions} is the conv-free case.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

namespace qac_b200 {

namespace returns {

struct Experience {  // returns.hpp:13-19
  std::vector<double> state;
  int action = 0;
  double reward = 0.0;
  double value_at_play = 0.0;
  std::uint64_t produced_version = 0;
};

struct ExperienceBatch {  // returns.hpp:21-26
  std::vector<Experience> experiences;
  std::vector<double> returns;
  bool terminal = false;
  int agent_id = 0;
};

// returns.hpp:31 / returns.cpp:8-26, computed on the device (fp64, bitwise).
std::vector<double> compute_returns(std::span<const double> rewards, bool terminal,
                                    double bootstrap_value, double gamma);

}  // namespace returns

namespace nnet {

struct ConvLayer {  // extension: VALID NHWC conv, OHWI weights
  int out = 0, k = 0, stride = 1;
};

struct NetworkSpec {  // nnet.hpp:14-18 (+ conv extension)
  int input_dim = 0;
  std::vector<int> hidden_dims;
  int n_actions = 0;
  // conv extension: input is in_h x in_w x (input_dim / (in_h*in_w)) NHWC
  int in_h = 1, in_w = 1;
  std::vector<ConvLayer> conv;
};

struct Hyperparams {  // nnet.hpp:20-31
  double gamma = 0.99;
  int t_max = 5;
  double beta = 0.01;
  double eps_log = 1e-6;
  double eta = 3e-4;
  double alpha = 0.99;
  double eps_rms = 1e-8;
  double value_loss_weight = 0.5;
  double grad_clip_norm = 0.0;
  bool clip_rewards = false;
};

struct ModelState {  // nnet.hpp:35-38
  std::vector<double> theta;
  std::uint64_t version = 0;
};

struct RmsState {  // nnet.hpp:41-43
  std::vector<double> g;
};

struct GradientPacket {  // nnet.hpp:47-53
  std::vector<double> dtheta;
  double policy_loss = 0.0;
  double value_loss = 0.0;
  double entropy = 0.0;
  int batch_size = 0;
};

struct ForwardResult {  // nnet.hpp:55-58
  std::vector<std::vector<double>> policies;
  std::vector<double> values;
};

struct UpdateResult {  // nnet.hpp:60-64
  ModelState model;
  RmsState rms;
  bool applied = false;
};

void validate(const NetworkSpec& spec);  // nnet.cpp:123-130
void validate(const Hyperparams& hp);    // nnet.cpp:131-145
std::size_t param_count(const NetworkSpec& spec);                     // nnet.hpp:71
ModelState init_model(const NetworkSpec& spec, std::uint64_t seed);   // nnet.hpp:75
RmsState init_rms(const NetworkSpec& spec);                           // nnet.hpp:77
ForwardResult forward(const ModelState& model, const NetworkSpec& spec,
                      std::span<const std::vector<double>> states);   // nnet.hpp:81-82
double policy_entropy(std::span<const double> policy, double eps_log);  // nnet.hpp:86
GradientPacket loss_and_gradients(const ModelState& model, const NetworkSpec& spec,
                                  const Hyperparams& hp,
                                  const returns::ExperienceBatch& batch);  // nnet.hpp:95-96
UpdateResult rmsprop_update(const ModelState& model, const RmsState& rms,
                            const GradientPacket& grads, const Hyperparams& hp);  // nnet.hpp:103-104

// The device this thread's calls run on (default 0).
void set_device(int device);

}  // namespace nnet
}  // namespace qac_b200
