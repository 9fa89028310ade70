// ORACLE — TEST INFRASTRUCTURE ONLY.
// Link-time stand-in for the one symbol the conv-path reference TUs pull in
// from the translation units that need Eigen decompositions (reduction.cpp):
// tg::lattice_sum_composite(..., reduce_eps) calls tg::reduce_rank.  The
// reference binary built here cannot run that branch; calling it throws.
#include <stdexcept>

#include "tengrid/reduction.hpp"

namespace tg {
CanonicalTensor3 reduce_rank(const CanonicalTensor3&, const ReductionConfig&) {
  throw std::logic_error("oracle/_ref: reduce_rank needs Eigen decompositions (reduction.cpp not built)");
}
}  // namespace tg
