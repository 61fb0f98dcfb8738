// host.hpp -- host-side input generation and preprocessing shared by every
// entry point of the library (not on the device path).
#pragma once
#include <cstdint>

namespace crb {
namespace host {

// xoshiro256++ named sub-stream normals (rng.hpp:41-59), row-major fill
void normal_stream(uint64_t seed, uint64_t tag, int64_t count, double* out, int max_threads = 16);
void uniform_pairs(uint64_t seed, uint64_t tag, int64_t count, double* out2);

}  // namespace host
}  // namespace crb
