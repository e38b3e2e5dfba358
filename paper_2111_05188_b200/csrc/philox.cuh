// philox.cuh — counter-based Philox4x32-10 (Salmon et al., SC'11) and the
// Box–Muller transform for the Gaussian action noise (R#14).
// counter = (env_global, step_lo, quad, step_hi), key = (seed_lo, seed_hi);
// ticker i uses quad i/4, component i%4.
#pragma once
#include <cstdint>

namespace pod {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

// Four standard normals from one Philox call (two Box–Muller pairs), float32:
// u1 = (x0 + 1) 2^-32 in (0, 1], u2 = x1 2^-32 in [0, 1),
// z0 = sqrt(-2 ln u1) cos(2 pi u2), z1 = sqrt(-2 ln u1) sin(2 pi u2).
// ln is the accurate logf (its argument approaches 1, where an approximate log's absolute
// error would be amplified by the square root); the square root and the sine/cosine use the
// SFU approximations (relative 2^-23; absolute 2^-20.9 on [0, 2 pi)), so |z - z_exact| <~ 1e-5,
// inside the parity tolerance 2e-5 |z| + 5e-4 (tests/test_gpu_parity.py).
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float4 normals4(uint64_t seed, uint32_t env_global, uint64_t step, uint32_t quad) {
    const uint4 x = philox4x32_10(make_uint4(env_global, static_cast<uint32_t>(step), quad,
                                             static_cast<uint32_t>(step >> 32)),
                                  make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)));
    const float s = 2.3283064365386963e-10f;  // 2^-32
    float4 z;
    {
        const float u1 = fmaf(__uint2float_rn(x.x), s, s);
        const float u2 = __uint2float_rn(x.y) * s;
        const float rad = sqrt_approx(fmaxf(-2.0f * logf(u1), 0.0f));
        float sn, cs;
        __sincosf(6.28318530717958647692f * u2, &sn, &cs);
        z.x = rad * cs;
        z.y = rad * sn;
    }
    {
        const float u1 = fmaf(__uint2float_rn(x.z), s, s);
        const float u2 = __uint2float_rn(x.w) * s;
        const float rad = sqrt_approx(fmaxf(-2.0f * logf(u1), 0.0f));
        float sn, cs;
        __sincosf(6.28318530717958647692f * u2, &sn, &cs);
        z.z = rad * cs;
        z.w = rad * sn;
    }
    return z;
}

}  // namespace pod
