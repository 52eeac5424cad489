// CodState (amm.hpp:35-69, amm.cpp:27-122) on the B200 -- placeholder until
// the factored-operator engine lands (C5).
#include "aero_common.cuh"
#include "engines.hpp"

namespace aero_b200 {
struct CodEngine::Impl {};
CodEngine::CodEngine(int, int, double, double, int64_t, uint64_t, uint64_t, int) : im_(nullptr) {
    throw InvalidInput("CodState: not yet available on the B200 path");
}
CodEngine::~CodEngine() { delete im_; }
void CodEngine::update_block(const double*, const double*, int64_t, const int64_t*, aero_event*) {}
void CodEngine::query(double*, double*) {}
void CodEngine::query_product(double*) {}
void CodEngine::info(int32_t*, int64_t*, int64_t*, int64_t*) const {}
}  // namespace aero_b200
