// Philox4x32-10 counter-based generator (Salmon et al., SC'11), the single
// source of randomness of the simulator: external Poisson drive, initial
// membrane voltages and the device graph generator.  Host and device builds
// share this header so the engine is reproducible on either side.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define NC_HD __host__ __device__ __forceinline__
#else
#define NC_HD inline
#endif

struct nc_u32x4 { uint32_t x, y, z, w; };

NC_HD void nc_mulhilo32(uint32_t a, uint32_t b, uint32_t* hi, uint32_t* lo) {
#ifdef __CUDA_ARCH__
  *lo = a * b;
  *hi = __umulhi(a, b);
#else
  uint64_t p = (uint64_t)a * (uint64_t)b;
  *lo = (uint32_t)p;
  *hi = (uint32_t)(p >> 32);
#endif
}

NC_HD nc_u32x4 nc_philox4x32_10(nc_u32x4 c, uint32_t k0, uint32_t k1) {
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    nc_mulhilo32(0xD2511F53u, c.x, &hi0, &lo0);
    nc_mulhilo32(0xCD9E8D57u, c.z, &hi1, &lo1);
    nc_u32x4 n;
    n.x = hi1 ^ c.y ^ k0;
    n.y = lo1;
    n.z = hi0 ^ c.w ^ k1;
    n.w = lo0;
    c = n;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// Counter-word tags separating the independent streams.
#define NC_TAG_DRIVE 0xD21E0001u
#define NC_TAG_VINIT 0x1417AB01u
#define NC_TAG_GAPS  0x6A950001u
#define NC_TAG_EDGEP 0xE06E0001u
