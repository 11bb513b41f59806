// paper_1905_08375_b200/csrc/expsum.cu — fast method 2 (1-D fractional,
// exponential-sum scans). Placeholder until the scan kernels land: the plan
// runs the GPU direct quadrature (method 0).
#include "plan.hpp"

namespace nlg {

void expsum_setup(Plan& P) { P.fast_method = 0; }
void expsum_apply(Plan& P, const double* u, double* out, cudaStream_t s) {
  launch_direct(P, u, out, nullptr, 0, nullptr, s);
}
void expsum_free(Plan&) {}

}  // namespace nlg
