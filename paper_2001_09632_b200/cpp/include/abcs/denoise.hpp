// denoise (denoise.cpp:96-109) for the B200 drop-in (mirrors abcs/denoise.hpp).
// Device path: "identity", "blur", and "dct_threshold" with 8x8 tiles on dims divisible by 4.
#pragma once
#include <cstdint>
#include <map>
#include <string>

#include "abcs/image.hpp"

namespace abcs {

struct DenoiserSpec {
  std::string name = "dct_threshold";
  std::map<std::string, double> params;
  double param(const std::string& key, double fallback) const {
    auto it = params.find(key);
    return it == params.end() ? fallback : it->second;
  }
};

PixelImage denoise(const DenoiserSpec& spec, const PixelImage& field, double sigma);
// Monte-Carlo divergence with a std::mt19937_64(seed) Rademacher probe (denoise.cpp:111-128)
double divergence(const DenoiserSpec& spec, const PixelImage& field, double sigma, double epsilon, uint64_t seed);

}  // namespace abcs
