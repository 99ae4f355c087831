// Forwarding header: the drop-in API lives in sewald_b200.hpp.
#pragma once
#include "sewald/sewald_b200.hpp"
