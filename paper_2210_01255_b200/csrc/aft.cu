// Fourier solve with free directions (d = 0, 1, 2). Placeholder until the
// zero-padded / upsampled path lands.
#include "engine.h"

namespace sewald_b200 {

struct FourierPlanAFT {};

void aft_solve(sewald_gpu_session*, const double*, bool) {
    throw EngineError(SEWALD_EINVAL, "d < 3 Fourier path not built yet");
}

void AftDeleter::operator()(FourierPlanAFT* p) const { delete p; }

}  // namespace sewald_b200
