// oracle/shim/extended_stub.cpp -- TEST INFRASTRUCTURE, not product code.
//
// The reference's extended-precision table path (proj/src/spectral_extended.cpp)
// needs Boost.Multiprecision, which is absent here.  It is only reached for
// Precision::Extended (spectral.cpp:110-111, 141-145; element.cpp:8), which the
// hot path never uses, so these two entry points throw sfem::Error like any
// other unsupported request.
#include "sfem/spectral.hpp"

namespace sfem::detail {

AssumptionReport assumption_report_extended(int, double) {
  fail("oracle/_ref: extended precision unavailable (Boost.Multiprecision absent)");
}

TablePrimariesT<double> build_primaries_extended(int, int, int, std::vector<std::string>*) {
  fail("oracle/_ref: extended precision unavailable (Boost.Multiprecision absent)");
}

}  // namespace sfem::detail
