// Process-wide kernel-choice switches (diagnostics and tests; defaults are
// the measured best). Each starts from its SEWALD_* environment variable and
// can be changed at run time through sewald_gpu_set_option (include/sewald_gpu.h),
// so one test process can pin every kernel family against the oracle.
#pragma once

#include "../../include/sewald_gpu.h"

namespace sewald_b200 {

// Current value of option `which` (SEWALD_OPT_*).
int option(int which);
// Set option `which`; returns false for an unknown option or value.
bool set_option(int which, int value);
// Incremented by every set_option: sessions drop kernel-specific orderings
// built under other settings.
int options_epoch();

}  // namespace sewald_b200
