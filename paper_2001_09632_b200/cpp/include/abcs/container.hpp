// The .abcs v1 measurement container for the B200 drop-in (mirrors abcs/container.hpp;
// container.cpp:58-149): packed / parsed on the GPU through libabcs_b200, byte-identical
// to the reference writer.
#pragma once
#include <filesystem>

#include "abcs/sensing.hpp"

namespace abcs {

void write_measurement_set(const MeasurementSet& ms, const std::filesystem::path& path);
MeasurementSet read_measurement_set(const std::filesystem::path& path);

}  // namespace abcs
