// modarith.cuh -- 64-bit modular arithmetic for RNS limbs (q < 2^61).
//
// __host__ __device__ so that the CPU unit test (tests/test_modarith.py builds
// a tiny host harness) checks exactly the code the kernels run.  On sm_100a
// every 64-bit multiply is emulated on the 32-bit IMAD pipe, so the choice of
// reduction matters: Shoup for multiplications by a known constant
// (twiddles, scalars), Barrett-128 for variable x variable products, and
// lazy 128-bit accumulation for sums of products (reduce once per chunk).
#pragma once
#include <stdint.h>

#ifndef __CUDACC__
#define __host__
#define __device__
#define __forceinline__ inline
#endif

#define VR_HD __host__ __device__ __forceinline__

namespace vr {

VR_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

struct u128 {
    uint64_t lo, hi;
};

VR_HD u128 mul_wide(uint64_t a, uint64_t b) {
    u128 r;
    r.lo = a * b;
    r.hi = mulhi64(a, b);
    return r;
}

VR_HD void add_to(u128 &acc, const u128 &x) {
    uint64_t lo = acc.lo + x.lo;
    acc.hi += x.hi + (lo < acc.lo);
    acc.lo = lo;
}

VR_HD void mac_to(u128 &acc, uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    // fused 64x64 -> 128 multiply-accumulate with carry chain
    uint64_t lo = a * b, hi = __umul64hi(a, b);
    asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(acc.lo), "+l"(acc.hi) : "l"(lo), "l"(hi));
#else
    add_to(acc, mul_wide(a, b));
#endif
}

// Per-prime constants.
struct Modulus {
    uint64_t q;
    uint64_t r_hi, r_lo;  // floor(2^128 / q) = r_hi * 2^64 + r_lo
};

VR_HD uint64_t add_mod(uint64_t a, uint64_t b, uint64_t q) {
    uint64_t s = a + b;
    return s >= q ? s - q : s;
}
VR_HD uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }
VR_HD uint64_t neg_mod(uint64_t a, uint64_t q) { return a ? q - a : 0; }

// Barrett reduction of a 128-bit value z (any z < 2^128) to [0, q).
// Quotient estimate floor(z * floor(2^128/q) / 2^128) is short of the true
// quotient by at most 2, so the remainder is < 3q < 2^64 before correction.
VR_HD uint64_t reduce128(u128 z, const Modulus &m) {
    uint64_t carry = mulhi64(z.lo, m.r_lo);
    u128 t = mul_wide(z.lo, m.r_hi);
    uint64_t mid = t.lo + carry;
    uint64_t c1 = t.hi + (mid < t.lo);
    u128 t2 = mul_wide(z.hi, m.r_lo);
    uint64_t mid2 = t2.lo + mid;
    uint64_t c2 = t2.hi + (mid2 < t2.lo);
    uint64_t qt = z.hi * m.r_hi + c1 + c2;
    uint64_t r = z.lo - qt * m.q;
    r = r >= m.q ? r - m.q : r;
    r = r >= m.q ? r - m.q : r;
    return r;
}

// x (< 2^64) mod q with a single-word Barrett.
VR_HD uint64_t reduce64(uint64_t x, const Modulus &m) {
    uint64_t qt = mulhi64(x, m.r_hi);
    uint64_t r = x - qt * m.q;
    r = r >= m.q ? r - m.q : r;
    r = r >= m.q ? r - m.q : r;
    return r;
}

VR_HD uint64_t mul_mod(uint64_t a, uint64_t b, const Modulus &m) { return reduce128(mul_wide(a, b), m); }

// Shoup: w_sh = floor(w * 2^64 / q).  Lazy variant returns [0, 2q) for any x < 2^64.
VR_HD uint64_t mul_shoup_lazy(uint64_t x, uint64_t w, uint64_t w_sh, uint64_t q) {
    uint64_t qh = mulhi64(x, w_sh);
    return x * w - qh * q;
}
VR_HD uint64_t mul_shoup(uint64_t x, uint64_t w, uint64_t w_sh, uint64_t q) {
    uint64_t r = mul_shoup_lazy(x, w, w_sh, q);
    return r >= q ? r - q : r;
}

// signed integer -> [0, q)
// Branch-free: a negative v is shifted by Q = q * floor(2^64 / q) (= q * r_hi, the largest
// multiple of q below 2^64), which keeps Q + v in [2^63 - q, 2^64) for every int64 v < 0.
VR_HD uint64_t from_i64(int64_t v, const Modulus &m) {
    const uint64_t x = (uint64_t)v + (v < 0 ? m.r_hi * m.q : 0);
    return reduce64(x, m);
}

// centered lift of x in [0, from) into [0, m.q)
VR_HD uint64_t lift_centered(uint64_t x, uint64_t from, const Modulus &m) {
    if (x > (from >> 1)) {
        uint64_t r = reduce64(from - x, m);
        return r ? m.q - r : 0;
    }
    return reduce64(x, m);
}

// ---- counter-based RNG (SplitMix64 finaliser), identical to the oracle ----
VR_HD uint64_t fmix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
VR_HD uint64_t stream_key(uint64_t seed, uint64_t dom, uint64_t a, uint64_t b) {
    uint64_t k = fmix64(seed ^ (dom * 0x9E3779B97F4A7C15ull));
    k = fmix64(k ^ (a * 0xC2B2AE3D27D4EB4Full));
    k = fmix64(k ^ (b * 0x165667B19E3779F9ull));
    return k;
}
VR_HD uint64_t rnd(uint64_t key, uint64_t i) { return fmix64(key + (i + 1) * 0x9E3779B97F4A7C15ull); }
VR_HD int64_t sample_ternary(uint64_t u) { return (int64_t)mulhi64(u, 3) - 1; }
VR_HD uint64_t sample_uniform(uint64_t u, uint64_t q) { return mulhi64(u, q); }

enum Domain : uint64_t {
    DOM_SK = 1, DOM_PK_A = 2, DOM_PK_E = 3, DOM_RLK_A = 4, DOM_RLK_E = 5,
    DOM_GAL_A = 6, DOM_GAL_E = 7, DOM_ENC_V = 8, DOM_ENC_E0 = 9, DOM_ENC_E1 = 10, DOM_ENC_A = 11
};

constexpr int CDT_LEN = 32;

}  // namespace vr
