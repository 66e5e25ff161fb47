// The reference's cut-posterior / fixed-location Sampler (mcmc.hpp), compiled
// UNCHANGED but with its LikelihoodWorkspace resolved to the B200 engine's
// drop-in (include/hawkes_b200/engine.hpp).  This is the integration a
// maintainer makes in engine.hpp; here it is done by name
// substitution so the reference sources stay untouched.
#include "hawkes/engine.hpp"
#include "hawkes_b200/engine.hpp"

namespace hawkes {
template <typename Real>
using LikelihoodWorkspaceB200 = b200::LikelihoodWorkspace<Real>;
}  // namespace hawkes

#define LikelihoodWorkspace LikelihoodWorkspaceB200
#define Sampler SamplerB200
#define run_cut_posterior run_cut_posterior_b200
#define run_fixed_posterior run_fixed_posterior_b200
#include "hawkes/mcmc.hpp"
#undef LikelihoodWorkspace
#undef Sampler
#undef run_cut_posterior
#undef run_fixed_posterior

namespace dropin {

hawkes::ChainOutput fixed_chain_b200(const hawkes::ChainConfig& config, const hawkes::Catalog& catalog) {
  return hawkes::run_fixed_posterior_b200(config, catalog);
}

hawkes::ChainOutput cut_chain_b200(const hawkes::ChainConfig& config, const hawkes::Catalog& catalog,
                                   const hawkes::RegionTable& regions) {
  return hawkes::run_cut_posterior_b200(config, catalog, regions);
}

}  // namespace dropin
