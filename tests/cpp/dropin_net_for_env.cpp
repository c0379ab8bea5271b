// cli::net_for_env (reference src/cli.cpp:161-168) for the drop-in builds:
// cli.cpp itself needs CLI11, which this image lacks, and the engine tests
// and the pybind module only need this one function from it.  Restated:
// the MLP's input and output widths come from a probe environment.
#include "qac/cli.hpp"

namespace qac::cli {

nnet::NetworkSpec net_for_env(const envs::EnvSpec& env, const std::vector<int>& hidden_dims) {
  const auto probe = envs::make_env(env);
  nnet::NetworkSpec spec;
  spec.input_dim = probe->observation_dim();
  spec.n_actions = probe->action_count();
  spec.hidden_dims = hidden_dims;
  return spec;
}

}  // namespace qac::cli
