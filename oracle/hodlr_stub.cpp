// oracle/hodlr_stub.cpp — link stub for the out-of-scope HODLR backend.
//
// TEST INFRASTRUCTURE ONLY. /root/reference/proj/src/operators.cpp:320-322
// references HodlrMatrix::compress/apply (SmoothBackend::Hodlr); hodlr.cpp needs
// Eigen's BDCSVD, which is absent. HODLR is out of scope, so the
// two symbols throw std::runtime_error if ever reached.
#include <stdexcept>

#include "nonloc/hodlr.hpp"

namespace nonloc {

HodlrMatrix HodlrMatrix::compress(const double*, std::int64_t, const HodlrOptions&) {
  throw std::runtime_error("HODLR backend is not built in the oracle (out of scope)");
}

std::vector<double> HodlrMatrix::apply(std::span<const double>) const {
  throw std::runtime_error("HODLR backend is not built in the oracle (out of scope)");
}

}  // namespace nonloc
