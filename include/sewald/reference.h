// Forwarding header: the analytic oracles (SPEC.md module `reference`) live in sewald_b200.hpp.
#pragma once
#include "sewald/sewald_b200.hpp"
