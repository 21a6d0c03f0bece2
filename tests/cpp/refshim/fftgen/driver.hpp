// tests/cpp/refshim/fftgen/driver.hpp -- the reference header path
// "fftgen/driver.hpp" mapped onto the B200 C++ API (test infrastructure).
#pragma once
#include "fftgen_b200.hpp"
