// Drop-in forwarding header: mpsgemm/tensor.hpp of the reference API
// (/root/reference/proj/include/mpsgemm/tensor.hpp) is provided by the B200
// implementation in ../mpsgemm_b200.hpp (namespace mpsgemm, libtcec_b200.so).
#pragma once
#include "../mpsgemm_b200.hpp"
