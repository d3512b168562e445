// denoise (denoise.cpp:96-109) for the B200 drop-in (mirrors abcs/denoise.hpp).
// Device path: "identity" and "dct_threshold" with 8x8 tiles on dims divisible by 4.
#pragma once
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

}  // namespace abcs
