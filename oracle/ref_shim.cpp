// ref_shim.cpp — TEST INFRASTRUCTURE ONLY. C entry points over the reference's own
// PhiloxRng (compiled from /root/reference/proj/core/src/rng.cpp by build_ref.sh) so the
// tests can pin the oracle's Philox restatement against the reference implementation.
#include <cstdint>
#include <sstream>
#include <cstring>

#include "mcmp2/rng.hpp"

extern "C" {
int ref_philox_block(const std::uint32_t* c, const std::uint32_t* k, std::uint32_t* out) {
  const auto o = mcmp2::PhiloxRng::block({c[0], c[1], c[2], c[3]}, {k[0], k[1]});
  for (int i = 0; i < 4; ++i) out[i] = o[i];
  return 0;
}
// kind 0: next_u32, 1: uniform, 2: gaussian3
int ref_philox_stream(std::uint64_t seed, std::uint32_t stream, int kind, int n, double* out) {
  mcmp2::PhiloxRng r(seed, stream);
  for (int i = 0; i < n; ++i) {
    if (kind == 0) out[i] = double(r.next_u32());
    else if (kind == 1) out[i] = r.uniform();
    else {
      const auto g = r.gaussian3();
      out[3 * i] = g[0]; out[3 * i + 1] = g[1]; out[3 * i + 2] = g[2];
    }
  }
  return 0;
}
// serialized state after `skip` u32 draws (rng.cpp:76-81)
int ref_philox_state(std::uint64_t seed, std::uint32_t stream, int skip, char* buf, int cap) {
  mcmp2::PhiloxRng r(seed, stream);
  for (int i = 0; i < skip; ++i) r.next_u32();
  std::ostringstream os;
  os << r;
  std::snprintf(buf, cap, "%s", os.str().c_str());
  return 0;
}
}
