// Internal helpers shared by the channel generators.
#pragma once
#include <cstdint>

namespace plb {

// In-place n-fold polar butterfly on an MSB-first packed bit word
// (code.cpp:12-31 semantics); the transform is its own inverse.
void polar_transform_words(uint64_t* w, int n);

} // namespace plb
