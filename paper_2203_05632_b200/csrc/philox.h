// philox.h — Philox4x32-10 and the reference's sequential stream, usable from host C++
// and device code (reference proj/core/src/rng.cpp:17-64).
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define MCMP2_HD __host__ __device__
#else
#define MCMP2_HD
#endif

namespace mcmp2dev {

// ------------------------------------------------------------------ Philox4x32-10
// Restates rng.cpp:17-39 (Random123 round + key schedule) for the device.
struct U32x4 {
  uint32_t v[4];
};

MCMP2_HD inline U32x4 philox_block(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                              uint32_t k0, uint32_t k1) {
#if defined(__CUDACC__)
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = uint64_t(0xD2511F53u) * c0;
    const uint64_t p1 = uint64_t(0xCD9E8D57u) * c2;
    const uint32_t n0 = uint32_t(p1 >> 32) ^ c1 ^ k0;
    const uint32_t n2 = uint32_t(p0 >> 32) ^ c3 ^ k1;
    c1 = uint32_t(p1);
    c3 = uint32_t(p0);
    c0 = n0;
    c2 = n2;
  }
  U32x4 o;
  o.v[0] = c0;
  o.v[1] = c1;
  o.v[2] = c2;
  o.v[3] = c3;
  return o;
}

// The reference stream of one worker: u32 number n of PhiloxRng(seed, stream) is word n%4
// of block n/4, block index = the 96-bit counter (rng.cpp:46-51) with word 3 = stream.
// `pos` addresses u32 draws directly, so every walker can start at its own offset.
struct StreamReader {
  uint32_t k0, k1, stream;
  uint64_t pos;
  uint64_t cached_block;
  U32x4 buf;
  MCMP2_HD StreamReader(uint32_t k0_, uint32_t k1_, uint32_t s_, uint64_t pos_)
      : k0(k0_), k1(k1_), stream(s_), pos(pos_), cached_block(~uint64_t(0)) {
#if !defined(__CUDA_ARCH__)
    buf = U32x4{{0u, 0u, 0u, 0u}};  // host: never read before the first refill; keeps -Wall quiet
#endif
  }
  MCMP2_HD uint32_t next_u32() {
    const uint64_t b = pos >> 2;
    if (b != cached_block) {
      buf = philox_block(uint32_t(b), uint32_t(b >> 32), 0u, stream, k0, k1);
      cached_block = b;
    }
    const unsigned i = unsigned(pos & 3);  // select, not an indexed load (keeps buf in registers)
    const uint32_t v = i == 0 ? buf.v[0] : i == 1 ? buf.v[1] : i == 2 ? buf.v[2] : buf.v[3];
    ++pos;
    return v;
  }
  // rng.cpp:58-64
  MCMP2_HD double uniform() {
    const uint64_t hi = next_u32();
    const uint64_t lo = next_u32();
    return double(((hi << 32) | lo) >> 11) * 0x1.0p-53;
  }
};

}  // namespace mcmp2dev
