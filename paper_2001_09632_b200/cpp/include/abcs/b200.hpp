// B200 device-path extras of the drop-in shim: the error for features outside the
// device path, and device selection. The shim keeps one libabcs_b200 context per
// host thread on the current CUDA device.
#pragma once
#include <stdexcept>
#include <string>

namespace abcs {

// A reference feature the device path does not implement (e.g. ISTA/AMP/DAMP, the blur
// denoiser, non-integer pixel values). Derives from std::logic_error so callers that
// catch the reference's exception hierarchy still see it.
class UnsupportedError : public std::logic_error {
 public:
  using std::logic_error::logic_error;
};

namespace b200 {
// CUDA device the calling thread's shim context uses (default: the current device).
void set_device(int device);
int device();
// Kernels launched so far by the calling thread's context.
long long launch_count();
}  // namespace b200

}  // namespace abcs
