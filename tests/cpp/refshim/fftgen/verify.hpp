// tests/cpp/refshim/fftgen/verify.hpp -- "fftgen/verify.hpp" mapped onto
// include/fftgen_b200_verify.hpp (test infrastructure).
#pragma once
#include "fftgen_b200_verify.hpp"
