// ntt_impl.cuh -- batched negacyclic NTT / INTT kernels with fused prologues
// and epilogues (included by ntt.cu and keyswitch.cu).
//
// Transform definition (identical to oracle/ckks_oracle.c orc_ntt/orc_intt):
//   forward  = Cooley-Tukey, natural in -> bit-reversed out; stage g pairs
//              elements at distance N >> (g+1) with twiddle
//              psi_br[2^g + (E >> (logN - g))]  (E = index of the upper element);
//   inverse  = Gentleman-Sande with psi^-1 in the same indexing, times N^-1.
//
// Structure.  N = N1 * N2.  Pass 1 runs stages g < log N1 on "columns"
// {c + r*N2}; a CTA stages TPC adjacent columns (coalesced rows).  Pass 2 runs
// the remaining stages inside contiguous N2-element rows.  Each thread owns 8
// elements and performs up to three stages per radix-8 group in registers;
// groups exchange through (swizzled) shared memory.  The group schedule is a
// compile-time function of the tile size, so every index is constant-folded.
// Butterflies are Harvey-lazy (forward values in [0,4q), inverse [0,2q)) with
// Shoup twiddle products; twiddles and their Shoup companions are stored
// interleaved so each butterfly issues one 16-byte load.  The inverse folds
// N^-1 into its last stage.
//
// Fusion.  The first pass reads its input through a Load functor and the last
// pass writes through a Store functor, so base conversions (centred lift from
// another prime), pointer-table gathers and the ModDown / rescale combine
// "(a - z) * q^-1" run inside the transform instead of as separate kernels.
#pragma once
#include <cstdlib>
#include <type_traits>
#include "vrhe_internal.cuh"

#include <cooperative_groups.h>

namespace vr {
namespace nttk {

__device__ __forceinline__ bool locate(const NttBatch &b, int t, int N, uint64_t *&ptr, int &pidx) {
    const int g = t / b.group, r = t - g * b.group;
    if (b.skip_diag > 0 && r == g % b.skip_diag) return false;
    ptr = (t < b.split ? b.data + (long long)g * b.gstride : b.data2 + (long long)(g - b.split / b.group) * b.gstride) +
          (long long)r * N;
    pidx = r < b.nq ? b.poff + r : b.pspecial;
    return true;
}

template <bool COLS>
__device__ __forceinline__ int sidx(int j, int L, int T, int TPC) {
    if (COLS) return L * TPC + j;
    return j * T + (L ^ ((L >> 4) & 15));
}
// The row swizzle sw(L) = L ^ ((L >> 4) & 15) is linear over GF(2), so for an element
// L = base | c (disjoint bits, c a compile-time constant) sw(L) = sw(base) ^ sw(c); with the row
// offset j*T above every swizzled bit, the index is (j*T | sw(base)) ^ sw(c): one XOR per access.
__host__ __device__ constexpr int swz(int L) { return L ^ ((L >> 4) & 15); }
template <bool COLS>
__device__ __forceinline__ int sidx_base(int j, int base, int T, int TPC) {
    if (COLS) return base * TPC + j;
    return (j * T) | swz(base);
}
template <bool COLS>
__device__ __forceinline__ int sidx_off(int sb, int c, int TPC) {
    if (COLS) return sb + c * TPC;
    return sb ^ swz(c);
}

__device__ __forceinline__ void bf_fwd(uint64_t &X, uint64_t &Y, ulonglong2 w, uint64_t q, uint64_t q2) {
    const uint64_t x = X >= q2 ? X - q2 : X;
    const uint64_t t = mul_shoup_lazy(Y, w.x, w.y, q);
    X = x + t;
    Y = x - t + q2;
}

__device__ __forceinline__ void bf_inv(uint64_t &X, uint64_t &Y, ulonglong2 w, uint64_t q, uint64_t q2) {
    uint64_t t = X + Y;
    t = t >= q2 ? t - q2 : t;
    const uint64_t u = X - Y + q2;
    Y = mul_shoup_lazy(u, w.x, w.y, q);
    X = t;
}

// ---- functor plumbing ---------------------------------------------------------
// A Load functor is `uint64_t operator()(ptr, t, E, primes, pidx)`.  A functor whose per-element
// work depends on the transform (row pointers, the source prime, constants behind integer divisions
// of t) may instead expose `Prep prep(t, primes, pidx)` -- evaluated once per thread -- and
// `uint64_t load(const Prep &, E)`: the element loads are then straight-line and issue together.
// Store functors likewise: either prefetch(t, E, ..) / finish(ptr, t, E, v, pre, ..), or
// `Ctx ctx(ptr, t, primes, pidx)` with prefetch(ctx, E) / finish(ctx, E, v, pre).
struct NoPrep {};
template <class F, class = void>
struct has_prep : std::false_type {};
template <class F>
struct has_prep<F, std::void_t<typename F::Prep>> : std::true_type {};
template <class F, class = void>
struct has_ctx : std::false_type {};
template <class F>
struct has_ctx<F, std::void_t<typename F::Ctx>> : std::true_type {};

template <class LD>
__device__ __forceinline__ auto ld_prep(const LD &ld, int t, const DevPrimes &pr, int pidx) {
    if constexpr (has_prep<LD>::value) return ld.prep(t, pr, pidx);
    else return NoPrep{};
}
template <class LD, class P>
__device__ __forceinline__ uint64_t ld_at(const LD &ld, const P &p, const uint64_t *ptr, int t, long long E,
                                          const DevPrimes &pr, int pidx) {
    if constexpr (has_prep<LD>::value) return ld.load(p, E);
    else return ld(ptr, t, E, pr, pidx);
}
template <class ST>
__device__ __forceinline__ auto st_ctx(const ST &st, uint64_t *ptr, int t, const DevPrimes &pr, int pidx) {
    if constexpr (has_ctx<ST>::value) return st.ctx(ptr, t, pr, pidx);
    else return NoPrep{};
}
template <class ST, class C>
__device__ __forceinline__ typename ST::Pre st_pre(const ST &st, const C &c, int t, long long E, const DevPrimes &pr, int pidx) {
    if constexpr (has_ctx<ST>::value) return st.prefetch(c, E);
    else return st.prefetch(t, E, pr, pidx);
}
template <class ST, class C>
__device__ __forceinline__ void st_fin(const ST &st, const C &c, uint64_t *ptr, int t, long long E, uint64_t v,
                                       const typename ST::Pre &pre, const DevPrimes &pr, int pidx) {
    if constexpr (has_ctx<ST>::value) st.finish(c, E, v, pre);
    else st.finish(ptr, t, E, v, pre, pr, pidx);
}

// ---- load functors (first pass of a transform) -----------------------------
struct LdPlain {
    __device__ __forceinline__ uint64_t operator()(const uint64_t *ptr, int, long long E, const DevPrimes &, int) const {
        return ptr[E];
    }
};
// centred lift of src[(t / div) * N + E] from prime (from_fixed >= 0 ? from_fixed : (t/div) % mod) into the target prime
// When source and target primes both run the FP64 body (Ctx::f64mask), the FP64 transform takes
// any integer input below 2^51, so the centred lift needs no reduction: x - q_src is represented
// as x + liftk[src][dst] with liftk = q_dst * ceil(q_src / q_dst) - q_src (< q_dst), an exact
// non-negative value congruent to x - q_src.
struct LdLift {
    const uint64_t *src;
    int div, mod, from_fixed, N;
    uint64_t f64mask;
    const uint64_t *liftk;  // [MAXP][MAXP]: q_dst ceil(q_src / q_dst) - q_src
    const NttConst *ncs;
    // mode 0: x + (neg ? k : 0) -- both primes on the FP64 body (any integer below 2^51 enters the
    //         transform), or q_src <= q_dst (then k = q_dst - q_src and the result is canonical);
    // mode 1: a 60-bit source into an FP64-body prime: x = xh 2^32 + xl == xh (2^32 mod q) + xl, the
    //         product reduced on the FP64 pipe (|.| <= q), shifted by q to stay non-negative (< 2^51);
    // mode 2: the integer centred lift (one Barrett reduction), branch-free.
    struct Prep {
        const uint64_t *row;
        uint64_t from, half, k, q, r_hi;
        double qd, qinv, c32;
        int mode;
    };
    __device__ __forceinline__ Prep prep(int t, const DevPrimes &pr, int pidx) const {
        const int row = t / div;
        const int fp = from_fixed >= 0 ? from_fixed : row % mod;
        Prep p;
        p.row = src + (long long)row * N;
        p.from = pr.m[fp].q;
        p.half = p.from >> 1;
        p.k = liftk[fp * MAXP + pidx];
        p.q = pr.m[pidx].q;
        p.r_hi = pr.m[pidx].r_hi;
        const bool dst64 = (f64mask >> pidx) & 1ull;
        p.mode = (((f64mask >> fp) & 1ull) && dst64) || p.from <= p.q ? 0 : (dst64 ? 1 : 2);  // uniform over the CTA
        if (p.mode == 1) {
            const NttConst nc = ncs[pidx];
            p.qd = nc.qd;
            p.qinv = nc.qinv;
            p.c32 = nc.c32;
        } else {
            p.qd = p.qinv = p.c32 = 0.0;
        }
        return p;
    }
    __device__ __forceinline__ uint64_t load(const Prep &p, long long E) const;
};
// ptrs[t / div] + (t % div) * stride + off + E
struct LdGather {
    const uint64_t *const *ptrs;
    int div;
    long long stride, off;
    struct Prep {
        const uint64_t *p;
    };
    __device__ __forceinline__ Prep prep(int t, const DevPrimes &, int) const {
        const int a = t / div;
        return Prep{ptrs[a] + (long long)(t - a * div) * stride + off};
    }
    __device__ __forceinline__ uint64_t load(const Prep &p, long long E) const { return p.p[E]; }
};

// ---- store functors (last pass) ------------------------------------------------
// Store functors expose prefetch(t, E) -> Pre (all global loads the store needs) and
// finish(ptr, t, E, v, Pre): the kernel prefetches the 8 elements a thread owns before
// any store, so the loads are not serialised behind possibly-aliasing stores.
struct StPlain {
    struct Pre {};
    __device__ __forceinline__ Pre prefetch(int, long long, const DevPrimes &, int) const { return Pre{}; }
    __device__ __forceinline__ void finish(uint64_t *ptr, int, long long E, uint64_t v, const Pre &, const DevPrimes &,
                                           int) const {
        ptr[E] = v;
    }
};
// t = row * nout + i;  row = r0 * rdiv + r1:
//   out = (A[r0][(r1 * a_limbs + i) * N + E] - v) * inv_i  (+ add[r0][(r1 * nout + i) * N + perm_g(E)] if r1 < add_polys)
//   written to O[r0][(r1 * nout + i) * N + E]
struct StCombine {
    const uint64_t *const *A;
    uint64_t *const *O;
    const uint64_t *const *add;
    const uint64_t *inv;  // inv_tab row: (inv, shoup) pairs per target prime
    int nout, rdiv, a_limbs, add_polys, logN;
    uint32_t g;
    // hoisted rotations batched over amounts: output r0 = c * add_div + r adds add[c] permuted by gs_rows[r]
    const uint32_t *gs_rows = nullptr;
    int add_div = 1;
    struct Pre {
        uint64_t a, b;
    };
    struct Ctx {
        const uint64_t *a, *add;  // add == nullptr: nothing to add
        uint64_t *o;
        uint64_t inv, inv_sh, q;
        uint32_t g;
    };
    __device__ __forceinline__ Ctx ctx(uint64_t *, int t, const DevPrimes &pr, int pidx) const {
        const long long N = 1ll << logN;
        const int row = t / nout, i = t - row * nout;
        const int r0 = row / rdiv, r1 = row - r0 * rdiv;
        Ctx c;
        c.a = A[r0] + ((long long)r1 * a_limbs + i) * N;
        c.o = O[r0] + ((long long)r1 * nout + i) * N;
        c.add = nullptr;
        c.g = 1;
        if (add && r1 < add_polys) {
            const int ra = r0 / add_div;
            c.g = gs_rows ? gs_rows[r0 - ra * add_div] : g;
            c.add = add[ra] + ((long long)r1 * nout + i) * N;
        }
        c.inv = inv[2 * i];
        c.inv_sh = inv[2 * i + 1];
        c.q = pr.m[pidx].q;
        return c;
    }
    __device__ __forceinline__ Pre prefetch(const Ctx &c, long long E) const {
        Pre p;
        p.a = c.a[E];
        p.b = 0;
        if (c.add) {
            long long src = E;
            if (c.g != 1) {
                const uint32_t brk = __brev((uint32_t)E) >> (32 - logN);
                const uint32_t e = ((2u * brk + 1u) * c.g) & ((2u << logN) - 1u);
                src = (long long)(__brev((e - 1u) >> 1) >> (32 - logN));
            }
            p.b = c.add[src];
        }
        return p;
    }
    __device__ __forceinline__ void finish(const Ctx &c, long long E, uint64_t v, const Pre &p) const {
        uint64_t r = mul_shoup(sub_mod(p.a, v, c.q), c.inv, c.inv_sh, c.q);
        if (c.add) r = add_mod(r, p.b, c.q);
        c.o[E] = r;
    }
};

struct PassArgs {
    int logN, s0, TPC;
    int last;     // this pass writes the final (fully reduced) output through the store functor
    int raw_in;   // input is the other pass's intermediate (FP64 body: raw double bits)
    int raw_out;  // output is an intermediate for the other pass
    int prefetch = 0;  // pull this CTA's twiddles into L2 before the PDL wait (small latency-bound batches)
};

// Index algebra shared by every caller: a unit's elements sit at base | (w << log2(d)), w < 2^R,
// where base has no bits in [log2 d, log2 d + R).  So (base + w d) >> shift splits into
// (base >> shift) + (w >> (R - r)) for every stage r (shift = log2 d + R - r): one runtime twiddle
// address per stage, the w part a compile-time offset in the load's immediate.
template <bool INV, int R, int EPT>
__device__ __forceinline__ void group_compute(uint64_t (&x)[EPT], const int (&base)[EPT], int d, int s, int logT, int s0,
                                              int hi, uint64_t q, const ulonglong2 *__restrict__ W, const NttConst &nc) {
    constexpr int E2 = 1 << R, U = EPT >> R;
    const uint64_t q2 = 2 * q;
#pragma unroll
    for (int v = 0; v < U; v++) {
        // all twiddles of this unit first (independent loads in flight)
        ulonglong2 tw[E2 - 1];
#pragma unroll
        for (int r = 0, n = 0; r < R; r++) {
            const int g = s0 + s + r, half = E2 >> (r + 1), shift = logT - (s + r);
#pragma unroll
            for (int w = 0; w < E2; w += 2 * half, n++) {
                if (INV && g == 0) continue;
                tw[n] = __ldg(W + ((1 << g) + (hi << (g - s0)) + (base[v] >> shift)) + (w >> (R - r)));
            }
        }
#pragma unroll
        for (int rr = 0; rr < R; rr++) {
            const int r = INV ? R - 1 - rr : rr;
            const int g = s0 + s + r, half = E2 >> (r + 1);
            const int n0 = (1 << r) - 1;  // twiddle slots used by stage r start here
#pragma unroll
            for (int w = 0; w < E2; w++) {
                if (w & half) continue;
                uint64_t &X = x[v * E2 + w], &Y = x[v * E2 + w + half];
                if (INV && g == 0) {
                    const uint64_t a = X, b = Y;
                    X = mul_shoup_lazy(a + b, nc.ninv, nc.ninv_sh, q);
                    Y = mul_shoup_lazy(a - b + q2, nc.w0n, nc.w0n_sh, q);
                } else {
                    const ulonglong2 t = tw[n0 + w / (2 * half)];
                    if (INV) bf_inv(X, Y, t, q, q2);
                    else bf_fwd(X, Y, t, q, q2);
                }
            }
        }
    }
}

// ---- FP64-pipe arithmetic (primes q < 2^46; NttConst::f64) ------------------------------------
// Values are exact integers held in doubles.  t = y*w mod q is computed Shoup-style on the FP64
// pipe: h = fl(y w), l = y w - h (exact, FMA), qt = rint(h / q) (FMA with 1.5*2^52), and
// r = (h - qt q) + l, exact because h - qt q is an integer of magnitude <= 0.75 q; |r| <= q
// whenever |y| < 2^51.  Forward stages therefore grow |x| by at most q each (<= 17 q after 16
// stages), Gentleman-Sande stages fold their sums; every transform ends with a canonical
// reduction to [0, q), so the output residues are exactly those of the integer path.
constexpr double kF64Magic = 6755399441055744.0;  // 1.5 * 2^52
constexpr double kTwo52 = 4503599627370496.0;

__device__ __forceinline__ double u2d(uint64_t v) {  // v < 2^52
    return __dadd_rn(__longlong_as_double((long long)(v | 0x4330000000000000ull)), -kTwo52);
}
__device__ __forceinline__ uint64_t d2u(double x) {  // integer x in [0, 2^52)
    return (uint64_t)__double_as_longlong(__dadd_rn(x, kTwo52)) & 0x000FFFFFFFFFFFFFull;
}
__device__ __forceinline__ double rint_f(double x, double qinv) {
    return __dadd_rn(__fma_rn(x, qinv, kF64Magic), -kF64Magic);
}
__device__ __forceinline__ double mulmod_f(double y, double w, double q, double qinv) {
    const double h = __dmul_rn(y, w);
    const double l = __fma_rn(y, w, -h);
    return __dadd_rn(__fma_rn(-rint_f(h, qinv), q, h), l);
}
__device__ __forceinline__ double fold_f(double x, double q, double qinv) { return __fma_rn(-rint_f(x, qinv), q, x); }
__device__ __forceinline__ uint64_t canon_f(double x, double q, double qinv) {
    double r = fold_f(x, q, qinv);
    r = r < 0.0 ? __dadd_rn(r, q) : r;
    return d2u(r);
}

__device__ __forceinline__ uint64_t LdLift::load(const Prep &p, long long E) const {
    const uint64_t x = p.row[E];
    const bool neg = x > p.half;
    if (p.mode == 0) return neg ? x + p.k : x;
    if (p.mode == 1) {
        const double hi = mulmod_f(u2d(x >> 32), p.c32, p.qd, p.qinv);
        const double lo = __dadd_rn(u2d(x & 0xffffffffull), neg ? u2d(p.k) : 0.0);
        return d2u(__dadd_rn(__dadd_rn(hi, lo), p.qd));
    }
    const uint64_t y = neg ? p.from - x : x;
    uint64_t r = y - mulhi64(y, p.r_hi) * p.q;
    r = r >= p.q ? r - p.q : r;
    r = r >= p.q ? r - p.q : r;
    return neg ? (r ? p.q - r : 0) : r;
}

template <bool INV, int R, int EPT>
__device__ __forceinline__ void group_compute_f(double (&x)[EPT], const int (&base)[EPT], int d, int s, int logT, int s0,
                                                int hi, const double *__restrict__ W, const NttConst &nc) {
    constexpr int E2 = 1 << R, U = EPT >> R;
    const double q = nc.qd, qinv = nc.qinv;
#pragma unroll
    for (int v = 0; v < U; v++) {
        double tw[E2 - 1];
        // Stage s + r of the group reads 2^r twiddles at consecutive table indices starting at a
        // multiple of 2^r (base has no bits below the group's span and g - s0 >= r), so the two
        // twiddles of the second stage and the four of the third arrive as 16-byte loads: 4 loads per
        // radix-8 group instead of 7.
        auto twp = [&](int r) { return W + ((1 << (s0 + s + r)) + (hi << (s + r)) + (base[v] >> (logT - (s + r)))); };
        if (!(INV && s0 + s == 0)) tw[0] = __ldg(twp(0));
        if constexpr (R >= 2) {
            const double2 t = __ldg(reinterpret_cast<const double2 *>(twp(1)));
            tw[1] = t.x;
            tw[2] = t.y;
        }
        if constexpr (R >= 3) {
            const double2 *p = reinterpret_cast<const double2 *>(twp(2));
            const double2 t0 = __ldg(p), t1 = __ldg(p + 1);
            tw[3] = t0.x;
            tw[4] = t0.y;
            tw[5] = t1.x;
            tw[6] = t1.y;
        }
#pragma unroll
        for (int rr = 0; rr < R; rr++) {
            const int r = INV ? R - 1 - rr : rr;
            const int g = s0 + s + r, half = E2 >> (r + 1);
            const int n0 = (1 << r) - 1;
#pragma unroll
            for (int w = 0; w < E2; w++) {
                if (w & half) continue;
                double &X = x[v * E2 + w], &Y = x[v * E2 + w + half];
                if (INV && g == 0) {
                    const double a = X, b = Y;
                    X = mulmod_f(__dadd_rn(a, b), nc.ninv_d, q, qinv);
                    Y = mulmod_f(__dsub_rn(a, b), nc.w0n_d, q, qinv);
                } else if (INV) {
                    // Lazy sums: a group starts with |x| <= q (folded sums and products of the previous
                    // group, or canonical input), each stage at most doubles a sum, so after R <= 3
                    // stages |x| <= 8q < 2^49 -- inside mulmod_f's |y| < 2^51 domain (its input a - b
                    // is bounded by the same sums).  Only the sums leaving the group are folded back
                    // to |x| <= q/2: 4 folds per 12 butterflies of a radix-8 group instead of 12.
                    const double a = X, b = Y;
                    X = rr == R - 1 ? fold_f(__dadd_rn(a, b), q, qinv) : __dadd_rn(a, b);
                    Y = mulmod_f(__dsub_rn(a, b), tw[n0 + w / (2 * half)], q, qinv);
                } else {
                    const double t = mulmod_f(Y, tw[n0 + w / (2 * half)], q, qinv);
                    const double a = X;
                    X = __dadd_rn(a, t);
                    Y = __dsub_rn(a, t);
                }
            }
        }
    }
}

// LE = log2(elements per thread): 3 (radix-8 groups) for throughput, 2 (radix-4 groups, twice the
// threads, half the per-thread dependency chain) for small latency-bound batches.
// The CTA's prime picks the integer (Harvey/Shoup, IMAD pipe) or the FP64-pipe body; a.raw_in /
// a.raw_out mark the intermediate between the two passes of one transform, which the FP64 body
// keeps as raw double bits (the integer body as lazy [0, 4q) residues).
template <bool INV, bool COLS, int LOGT, int LE, bool F64, class LD, class ST>
__device__ __forceinline__ void ntt_pass_body(const NttBatch &b, const PassArgs &a, const DevPrimes &pr,
                                              const ulonglong2 *__restrict__ tw, const double *__restrict__ twd,
                                              const NttConst &nc, uint64_t *ptr, int t, int pidx, const LD &ld,
                                              const ST &st, uint64_t *sm) {
    using V = typename std::conditional<F64, double, uint64_t>::type;
    constexpr int EPT = 1 << LE;
    constexpr int T = 1 << LOGT, NG = (LOGT + LE - 1) / LE;
    const int logN = a.logN, N = 1 << logN, s0 = a.s0;
    const int lo_bits = logN - s0 - LOGT, TPC = a.TPC;
    const int chunks = (N >> LOGT) / TPC;
    const int chunk = blockIdx.x - t * chunks;
    const uint64_t q = pr.m[pidx].q;
    const ulonglong2 *W = tw + (size_t)pidx * N;
    const double *Wd = twd + (size_t)pidx * N;
    const int tile0 = chunk * TPC, lomask = (1 << lo_bits) - 1;
    constexpr int tpt = T >> LE;
    int j, sub;
    if (COLS) { j = threadIdx.x % TPC; sub = threadIdx.x / TPC; }
    else { j = threadIdx.x / tpt; sub = threadIdx.x - j * tpt; }
    const int tile = tile0 + j, hi = tile >> lo_bits, lo = tile & lomask;
    const long long ebase = ((long long)hi << (logN - s0)) | lo;
    V *smv = reinterpret_cast<V *>(sm);
    const auto lprep = ld_prep(ld, t, pr, pidx);  // per-thread state of the fused load (dead after the loads)

    // element conversion at the pass boundaries
    auto in = [&](uint64_t u) -> V {
        if constexpr (F64) return a.raw_in ? __longlong_as_double((long long)u) : u2d(u);
        else return u;
    };
    auto out_final = [&](V v) -> uint64_t {
        if constexpr (F64) return canon_f(v, nc.qd, nc.qinv);
        else {
            const uint64_t q2 = 2 * q;
            uint64_t w = v;
            if (!INV) w = w >= q2 ? w - q2 : w;
            return w >= q ? w - q : w;
        }
    };
    auto out_raw = [&](V v) -> uint64_t {
        if constexpr (F64) return (uint64_t)__double_as_longlong(v);
        else return v;
    };

    V x[EPT];
    int base[EPT];
    const int wl = blockDim.x < 32 ? (int)blockDim.x : 32;
    const int own0 = ((int)threadIdx.x / wl) * (wl * EPT) + ((int)threadIdx.x % wl);  // warp-owned block, lane-contiguous
    // The inverse rows pass starts with its shortest-distance round, where a thread owns runs of
    // consecutive elements: loaded directly, every warp-wide load touches 32 sectors.  Stage the tile
    // through shared memory instead (lane-contiguous loads of the warp's own block, which is exactly
    // what that round reads, so __syncwarp orders it).
    constexpr bool STAGE_IN = INV && !COLS;
    if constexpr (STAGE_IN) {
        V y[EPT];
#pragma unroll
        for (int r = 0; r < EPT; r++) {
            const int idx = own0 + r * wl;
            const int jj = idx >> LOGT, mid = idx & (T - 1);
            const int tl = tile0 + jj, h2 = tl >> lo_bits, lo2 = tl & lomask;
            y[r] = in(ld_at(ld, lprep, ptr, t, ((long long)h2 << (logN - s0)) | ((long long)mid << lo_bits) | lo2, pr, pidx));
        }
#pragma unroll
        for (int r = 0; r < EPT; r++) {
            const int idx = own0 + r * wl;
            smv[sidx<COLS>(idx >> LOGT, idx & (T - 1), T, TPC)] = y[r];
        }
        __syncwarp();
    }
#pragma unroll
    for (int step = 0; step < NG; step++) {
        const int gi = INV ? NG - 1 - step : step;
        const int s = LE * gi, R = (LOGT - s) < LE ? (LOGT - s) : LE;
        const int logd = LOGT - s - R, d = 1 << logd, E2 = 1 << R;
#pragma unroll
        for (int v = 0; v < EPT; v++) {
            const int uid = sub * (EPT >> R) + v;
            base[v] = v < (EPT >> R) ? (((uid >> logd) << (logd + R)) | (uid & (d - 1))) : 0;
        }
        int sb[EPT];
#pragma unroll
        for (int v = 0; v < EPT; v++) sb[v] = sidx_base<COLS>(j, base[v], T, TPC);
#pragma unroll
        for (int e = 0; e < EPT; e++) {
            const int L = base[e >> R] | ((e & (E2 - 1)) << logd);
            if (step == 0 && !STAGE_IN) x[e] = in(ld_at(ld, lprep, ptr, t, ebase | ((long long)L << lo_bits), pr, pidx));
            else x[e] = smv[sidx_off<COLS>(sb[e >> R], (e & (E2 - 1)) << logd, TPC)];
        }
        if constexpr (F64) {
            if (R == 3) group_compute_f<INV, (LE >= 3 ? 3 : 1), EPT>(x, base, d, s, LOGT, s0, hi, Wd, nc);
            else if (R == 2) group_compute_f<INV, 2, EPT>(x, base, d, s, LOGT, s0, hi, Wd, nc);
            else group_compute_f<INV, 1, EPT>(x, base, d, s, LOGT, s0, hi, Wd, nc);
        } else {
            if (R == 3) group_compute<INV, (LE >= 3 ? 3 : 1), EPT>(x, base, d, s, LOGT, s0, hi, q, W, nc);
            else if (R == 2) group_compute<INV, 2, EPT>(x, base, d, s, LOGT, s0, hi, q, W, nc);
            else group_compute<INV, 1, EPT>(x, base, d, s, LOGT, s0, hi, q, W, nc);
        }
        const bool last_group = step == NG - 1;
        if (last_group && COLS) {
            // consecutive threads own consecutive columns -> coalesced direct stores
            const auto sctx = st_ctx(st, ptr, t, pr, pidx);  // built here: not live across the transform
            typename ST::Pre pre[EPT];
#pragma unroll
            for (int e = 0; e < EPT; e++) {
                const int L = base[e >> R] + (e & (E2 - 1)) * d;
                pre[e] = st_pre(st, sctx, t, ebase | ((long long)L << lo_bits), pr, pidx);
            }
#pragma unroll
            for (int e = 0; e < EPT; e++) {
                const int L = base[e >> R] + (e & (E2 - 1)) * d;
                const uint64_t v = a.last ? out_final(x[e]) : (a.raw_out ? out_raw(x[e]) : out_final(x[e]));
                st_fin(st, sctx, ptr, t, ebase | ((long long)L << lo_bits), v, pre[e], pr, pidx);
            }
            return;
        }
#pragma unroll
        for (int e = 0; e < EPT; e++) smv[sidx_off<COLS>(sb[e >> R], (e & (E2 - 1)) << logd, TPC)] = x[e];
        // One owner per element within a group: a single barrier per group boundary.  Rows passes: a
        // warp's 32 * EPT elements are one contiguous block of the flat tile array, and a round whose
        // span (2^(LOGT - s)) fits that block reads and writes only that block, so the exchange with the
        // next round (and with the warp-owned store below) never leaves the warp: __syncwarp, and the
        // warps of a CTA drift apart instead of meeting at every radix group.
        {
            constexpr int W = 32 * EPT;
            const int need = INV ? (gi > 0 ? (1 << (LOGT - LE * (gi - 1))) : T) : (1 << (LOGT - s));
            if (!COLS && need <= W) __syncwarp();
            else __syncthreads();
        }
    }
    // rows: coalesced store out of shared memory, each warp its own block (prefetch the epilogue's loads first)
    long long Es[EPT];
    typename ST::Pre pre[EPT];
    const auto sctx = st_ctx(st, ptr, t, pr, pidx);
#pragma unroll
    for (int r = 0; r < EPT; r++) {  // blockDim.x * EPT == TPC * T
        const int idx = own0 + r * wl;
        const int jj = idx >> LOGT, mid = idx & (T - 1);
        const int tl = tile0 + jj, h2 = tl >> lo_bits, lo2 = tl & lomask;
        Es[r] = ((long long)h2 << (logN - s0)) | ((long long)mid << lo_bits) | lo2;
        pre[r] = st_pre(st, sctx, t, Es[r], pr, pidx);
    }
#pragma unroll
    for (int r = 0; r < EPT; r++) {
        const int idx = own0 + r * wl;
        const int jj = idx >> LOGT, mid = idx & (T - 1);
        const V v = smv[sidx<COLS>(jj, mid, T, TPC)];
        st_fin(st, sctx, ptr, t, Es[r], a.last ? out_final(v) : (a.raw_out ? out_raw(v) : out_final(v)), pre[r], pr, pidx);
    }
}

// Register cap (64) on every transform kernel.  Uncapped, the integer and FP64 bodies sharing one
// kernel took 94-128 registers (inverse passes and fused-epilogue passes: 23-25% occupancy in ncu);
// capped, the fused epilogues spill up to ~250 B of prefetched operands to L1-resident local memory
// and still run faster: config 4 49.2 -> 52.1 images/s, the fused encryption NTT 110 -> 82 us.
constexpr int kCapRegs = 64;

// Pull the twiddles a pass's CTA will read into L2 before the PDL wait (the tables are constant,
// so this overlaps the previous kernel's tail).  Between the steps of a workload the streaming
// passes (the tensor sums read 250 MB per cfg-2 step) evict them, and the small latency-bound
// batches of a key switch otherwise pay one HBM round trip per radix group (cfg-2 chain 47.5 ->
// 44.8 us).  Only the small-batch (radix-4) passes do it: for large batches the twiddles stay in
// L2 and the extra instructions cost throughput (cfg 4 52.4 -> 47.7 images/s when unconditional).  Stage g of this CTA
// reads entries [2^g + h_lo 2^(g-s0), 2^g + (h_hi + 1) 2^(g-s0)) with h = tile >> lo_bits.
__device__ __forceinline__ void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
template <int LOGT>
__device__ __forceinline__ void prefetch_pass_twiddles(const PassArgs &a, const char *table, int esz, int tile0) {
    const int lo_bits = a.logN - a.s0 - LOGT;
    const long long hlo = tile0 >> lo_bits, hhi = (tile0 + a.TPC - 1) >> lo_bits;
#pragma unroll 1
    for (int s = 0; s < LOGT; s++) {
        const long long g0 = 1ll << (a.s0 + s);
        const long long l0 = ((g0 + (hlo << s)) * esz) >> 7, l1 = ((g0 + ((hhi + 1) << s)) * esz - 1) >> 7;
        for (long long l = l0 + threadIdx.x; l <= l1; l += blockDim.x) prefetch_l2(table + (l << 7));
    }
}

template <bool INV, bool COLS, int LOGT, int LE, class LD, class ST>
__global__ void __launch_bounds__(512, 65536 / (512 * kCapRegs)) ntt_pass(NttBatch b, PassArgs a, DevPrimes pr, const ulonglong2 *__restrict__ tw,
                                                const double *__restrict__ twd, const NttConst *__restrict__ ncs, LD ld,
                                                ST st) {
    extern __shared__ uint64_t sm[];
    constexpr int T = 1 << LOGT;
    const int N = 1 << a.logN;
    const int chunks = (N >> LOGT) / a.TPC;
    const int t = blockIdx.x / chunks;
    uint64_t *ptr;
    int pidx;
    const bool live = locate(b, t, N, ptr, pidx);  // batch metadata only (no global reads)
    if (live && a.prefetch) {
        const bool f64 = ncs[pidx].f64;  // constant table
        prefetch_pass_twiddles<LOGT>(a, f64 ? (const char *)(twd + (size_t)pidx * N) : (const char *)(tw + (size_t)pidx * N),
                                     f64 ? 8 : 16, ((int)blockIdx.x - t * chunks) * a.TPC);
    }
    pdl_wait();
    pdl_trigger();
    if (!live) return;
    const NttConst nc = ncs[pidx];
    (void)T;
    if (nc.f64) ntt_pass_body<INV, COLS, LOGT, LE, true>(b, a, pr, tw, twd, nc, ptr, t, pidx, ld, st, sm);
    else ntt_pass_body<INV, COLS, LOGT, LE, false>(b, a, pr, tw, twd, nc, ptr, t, pidx, ld, st, sm);
}

// one thread per transform for N <= 4 (slots = 2, test-only parameter sets)
template <bool INV, class LD, class ST>
__global__ void ntt_tiny(NttBatch b, int logN, DevPrimes pr, const ulonglong2 *__restrict__ tw, const NttConst *__restrict__ ncs,
                         LD ld, ST st) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= b.count) return;
    const int N = 1 << logN;
    uint64_t *ptr;
    int pidx;
    if (!locate(b, t, N, ptr, pidx)) return;
    const uint64_t q = pr.m[pidx].q;
    const ulonglong2 *w = tw + (size_t)pidx * N;
    uint64_t a[4];
    const auto lprep = ld_prep(ld, t, pr, pidx);
    const auto sctx = st_ctx(st, ptr, t, pr, pidx);
    // fused loads may hand the FP64 body unreduced representatives; this integer loop wants [0, q)
    for (int k = 0; k < N; k++) a[k] = reduce64(ld_at(ld, lprep, ptr, t, k, pr, pidx), pr.m[pidx]);
    if (!INV) {
        int tt = N;
        for (int m = 1; m < N; m <<= 1) {
            tt >>= 1;
            for (int i = 0; i < m; i++)
                for (int jx = 2 * i * tt; jx < 2 * i * tt + tt; jx++) {
                    const uint64_t u = a[jx], v = mul_shoup(a[jx + tt], w[m + i].x, w[m + i].y, q);
                    a[jx] = add_mod(u, v, q);
                    a[jx + tt] = sub_mod(u, v, q);
                }
        }
    } else {
        int tt = 1;
        for (int m = N; m > 1; m >>= 1) {
            const int h = m >> 1;
            for (int i = 0, j1 = 0; i < h; i++, j1 += 2 * tt)
                for (int jx = j1; jx < j1 + tt; jx++) {
                    const uint64_t u = a[jx], v = a[jx + tt];
                    a[jx] = add_mod(u, v, q);
                    a[jx + tt] = mul_shoup(sub_mod(u, v, q), w[h + i].x, w[h + i].y, q);
                }
            tt <<= 1;
        }
        const NttConst nc = ncs[pidx];
        for (int k = 0; k < N; k++) a[k] = mul_shoup(a[k], nc.ninv, nc.ninv_sh, q);
    }
    for (int k = 0; k < N; k++) st_fin(st, sctx, ptr, t, k, a[k], st_pre(st, sctx, t, k, pr, pidx), pr, pidx);
}

template <bool INV, bool COLS, int LOGT, int LE, class LD, class ST>
void launch_pass(Ctx &c, const NttBatch &b, const PassArgs &a, const LD &ld, const ST &st) {
    constexpr int T = 1 << LOGT;
    const int chunks = (c.n >> LOGT) / a.TPC;
    const int threads = a.TPC * (T >> LE);
    const size_t smem = (size_t)a.TPC * T * sizeof(uint64_t);
    const unsigned blocks = (unsigned)b.count * chunks;
    launch_pdl(ntt_pass<INV, COLS, LOGT, LE, LD, ST>, dim3(blocks), dim3(threads), smem, c.stream, b, a, c.primes,
               (const ulonglong2 *)(INV ? c.itw2 : c.tw2), (const double *)(INV ? c.itwd : c.twd),
               (const NttConst *)c.ntt_const, ld, st);
    check_launch("ntt_pass");
}

template <bool INV, bool COLS, class LD, class ST>
void dispatch_pass(Ctx &c, const NttBatch &b, const PassArgs &a, int logT, int le, const LD &ld, const ST &st) {
    if (le == 2 && logT >= 6 && logT <= 8) {
        switch (logT) {
            case 6: launch_pass<INV, COLS, 6, 2>(c, b, a, ld, st); return;
            case 7: launch_pass<INV, COLS, 7, 2>(c, b, a, ld, st); return;
            default: launch_pass<INV, COLS, 8, 2>(c, b, a, ld, st); return;
        }
    }
    switch (logT) {
        case 3: launch_pass<INV, COLS, 3, 3>(c, b, a, ld, st); break;
        case 4: launch_pass<INV, COLS, 4, 3>(c, b, a, ld, st); break;
        case 5: launch_pass<INV, COLS, 5, 3>(c, b, a, ld, st); break;
        case 6: launch_pass<INV, COLS, 6, 3>(c, b, a, ld, st); break;
        case 7: launch_pass<INV, COLS, 7, 3>(c, b, a, ld, st); break;
        case 8: launch_pass<INV, COLS, 8, 3>(c, b, a, ld, st); break;
        case 9: launch_pass<INV, COLS, 9, 3>(c, b, a, ld, st); break;
        case 10: launch_pass<INV, COLS, 10, 3>(c, b, a, ld, st); break;
        default: throw VrError(3, "unsupported NTT tile size");
    }
}

// Tiles per CTA: as many as fit a 512-thread CTA, reduced for small batches so
// the launch still spreads over every SM.
inline int pick_tpc(int count, int tiles_per_tf, int T, int max_tpc, int min_tpc, int le) {
    int tpc = max_tpc;
    while (tpc > min_tpc && (long long)count * (tiles_per_tf / tpc) < 2 * 148) tpc >>= 1;
    while (tpc > 1 && tpc * (T >> le) > 512) tpc >>= 1;
    if (tpc > tiles_per_tf) tpc = tiles_per_tf;
    return tpc;
}

// ---- one-kernel transform: a cluster of 8 CTAs per transform ------------------------------
// CTA r of the cluster owns the contiguous chunk [r C, (r+1) C), C = N / 8, in shared memory.
// Forward: the first three stages (distances N/2, N/4, N/8) pair elements {j + u C : u < 8}
// across the cluster: thread j of CTA r loads that column straight from global memory (through
// the Load functor), runs the three stages in registers and scatters element u into CTA u's
// shared memory (DSMEM).  The remaining log2(C) stages stay inside each chunk (radix-8 groups,
// exactly the rows pass of ntt_pass with s0 = 3), and the chunk leaves through the Store functor.
// Inverse: the local Gentleman-Sande stages first (input through the Load functor), then the
// last three stages gather each column from the eight CTAs.  One launch and one global round
// trip per transform instead of two.
__device__ __forceinline__ int sidx_row(int L) { return L ^ ((L >> 4) & 15); }

// DSMEM exchange with asynchronous stores (sm_90+): st.async writes a 64-bit value into a peer CTA's
// shared memory and completes transaction bytes on the peer's mbarrier, so a receiver waits only for
// the bytes addressed to it -- no release fence and no cluster-wide barrier after the scatter.
__device__ __forceinline__ uint32_t cl_smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cl_mapa(uint32_t a, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(cta));
    return r;
}
__device__ __forceinline__ void st_async_b64(uint32_t raddr, uint64_t v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr), "l"(v), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void cl_mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(cl_smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
inline bool cl_st_async() {
    static const bool on = [] {
        const char *e = getenv("VR_NTT_ST_ASYNC");
        return e == nullptr || atoi(e) != 0;
    }();
    return on;
}

template <bool INV, int LOGC, bool F64, class LD, class ST>
__device__ __forceinline__ void ntt_cl8_body(int logN, const DevPrimes &pr, const ulonglong2 *__restrict__ tw,
                                             const double *__restrict__ twd, const NttConst &nc, uint64_t *ptr, int t,
                                             int pidx, const LD &ld, const ST &st, uint64_t *sm, uint64_t *xbar, bool async_x) {
    namespace cg = cooperative_groups;
    using V = typename std::conditional<F64, double, uint64_t>::type;
    constexpr int LE = 3, EPT = 8, C = 1 << LOGC, NG = (LOGC + LE - 1) / LE;
    cg::cluster_group cluster = cg::this_cluster();
    const int r = (int)cluster.block_rank(), sub = threadIdx.x;
    const int N = 1 << logN;
    const uint64_t q = pr.m[pidx].q, q2 = 2 * q;
    const ulonglong2 *W = tw + (size_t)pidx * N;
    const double *Wd = twd + (size_t)pidx * N;
    const int col = r * (C / 8) + sub;  // this thread's cross-cluster column
    V *smv = reinterpret_cast<V *>(sm);
    V x[EPT];
    int base[EPT];
    const int zero_base[EPT] = {0, 0, 0, 0, 0, 0, 0, 0};
    const auto lprep = ld_prep(ld, t, pr, pidx);  // per-thread state of the fused load (dead after the loads)

    auto in = [&](uint64_t u) -> V {
        if constexpr (F64) return u2d(u);
        else return u;
    };
    auto final_value = [&](V v) -> uint64_t {
        if constexpr (F64) return canon_f(v, nc.qd, nc.qinv);
        else {
            uint64_t w = v;
            if (!INV) w = w >= q2 ? w - q2 : w;
            return w >= q ? w - q : w;
        }
    };
    auto compute = [&](auto rtag, int d, int s, int logT, int s0, int hi, const int(&bs)[EPT]) {
        constexpr int RR = decltype(rtag)::value;
        if constexpr (F64) group_compute_f<INV, RR, EPT>(x, bs, d, s, logT, s0, hi, Wd, nc);
        else group_compute<INV, RR, EPT>(x, bs, d, s, logT, s0, hi, q, W, nc);
    };
    auto local_stages = [&](bool from_global) {
        if (from_global) {  // inverse: coalesced loads of the warp-owned block, staged through shared memory
            const int own0 = (sub >> 5) * (32 * EPT) + (sub & 31);
            V y[EPT];
#pragma unroll
            for (int k = 0; k < EPT; k++) y[k] = in(ld_at(ld, lprep, ptr, t, (long long)r * C + own0 + 32 * k, pr, pidx));
#pragma unroll
            for (int k = 0; k < EPT; k++) smv[sidx_row(own0 + 32 * k)] = y[k];
            __syncwarp();
        }
#pragma unroll
        for (int step = 0; step < NG; step++) {
            const int gi = INV ? NG - 1 - step : step;
            const int s = LE * gi, R = (LOGC - s) < LE ? (LOGC - s) : LE;
            const int logd = LOGC - s - R, d = 1 << logd, E2 = 1 << R;
#pragma unroll
            for (int v = 0; v < EPT; v++) {
                const int uid = sub * (EPT >> R) + v;
                base[v] = v < (EPT >> R) ? (((uid >> logd) << (logd + R)) | (uid & (d - 1))) : 0;
            }
            int sb[EPT];
#pragma unroll
            for (int v = 0; v < EPT; v++) sb[v] = swz(base[v]);
#pragma unroll
            for (int e = 0; e < EPT; e++) x[e] = smv[sb[e >> R] ^ swz((e & (E2 - 1)) << logd)];
            if (R == 3) compute(std::integral_constant<int, 3>{}, d, s, LOGC, 3, r, base);
            else if (R == 2) compute(std::integral_constant<int, 2>{}, d, s, LOGC, 3, r, base);
            else compute(std::integral_constant<int, 1>{}, d, s, LOGC, 3, r, base);
#pragma unroll
            for (int e = 0; e < EPT; e++) smv[sb[e >> R] ^ swz((e & (E2 - 1)) << logd)] = x[e];
            // warp-owned 256-element blocks once a round's span fits them (see ntt_pass_body): only the
            // chunk-wide first round (forward) / last round and the peer exchange (inverse) meet CTA-wide
            {
                constexpr int W = 32 * EPT;
                const int need = INV ? (gi > 0 ? (1 << (LOGC - LE * (gi - 1))) : C) : (1 << (LOGC - s));
                if (need <= W) __syncwarp();
                else __syncthreads();
            }
        }
    };

    if (!INV) {
#pragma unroll
        for (int u = 0; u < 8; u++) x[u] = in(ld_at(ld, lprep, ptr, t, (long long)col + ((long long)u << LOGC), pr, pidx));
        compute(std::integral_constant<int, 3>{}, 1, 0, 3, 0, 0, zero_base);
        asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // every peer is resident (and its barrier set up)
        if (async_x) {
            if (threadIdx.x == 0)  // this CTA receives its whole chunk: C words from the 8 ranks
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(cl_smem_u32(xbar)), "r"((uint32_t)C * 8)
                             : "memory");
            const uint32_t dst = cl_smem_u32(&smv[sidx_row(col)]), bar = cl_smem_u32(xbar);
#pragma unroll
            for (int u = 0; u < 8; u++) {
                uint64_t bits;
                if constexpr (F64) bits = (uint64_t)__double_as_longlong(x[u]);
                else bits = x[u];
                st_async_b64(cl_mapa(dst, u), bits, cl_mapa(bar, u));
            }
            cl_mbar_wait(xbar, 0);
        } else {
#pragma unroll
            for (int u = 0; u < 8; u++) cluster.map_shared_rank(smv, u)[sidx_row(col)] = x[u];
            cluster.sync();
        }
        local_stages(false);
        // coalesced store of the chunk through the Store functor (prefetch its loads first)
        typename ST::Pre pre[EPT];
        const auto sctx = st_ctx(st, ptr, t, pr, pidx);
        const int own0 = (sub >> 5) * (32 * EPT) + (sub & 31);  // each warp stores the block it owns
#pragma unroll
        for (int k = 0; k < EPT; k++) pre[k] = st_pre(st, sctx, t, (long long)r * C + own0 + 32 * k, pr, pidx);
#pragma unroll
        for (int k = 0; k < EPT; k++) {
            const int mid = own0 + 32 * k;
            st_fin(st, sctx, ptr, t, (long long)r * C + mid, final_value(smv[sidx_row(mid)]), pre[k], pr, pidx);
        }
    } else {
        local_stages(true);
        if (async_x) {
            // push instead of gather: CTA u's thread `sub` needs element sidx_row(u C/8 + sub) of every
            // rank; it lands in u's receive buffer (behind its chunk) at [rank][sub]
            V *rx = smv + C;
            asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // peers resident, barriers set up
            if (threadIdx.x == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(cl_smem_u32(xbar)), "r"((uint32_t)C * 8)
                             : "memory");
            const uint32_t dst = cl_smem_u32(&rx[r * (C / 8) + sub]), bar = cl_smem_u32(xbar);
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const V v = smv[sidx_row(u * (C / 8) + sub)];
                uint64_t bits;
                if constexpr (F64) bits = (uint64_t)__double_as_longlong(v);
                else bits = v;
                st_async_b64(cl_mapa(dst, u), bits, cl_mapa(bar, u));
            }
            cl_mbar_wait(xbar, 0);
#pragma unroll
            for (int u = 0; u < 8; u++) x[u] = rx[u * (C / 8) + sub];
        } else {
            asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
            cluster.sync();
#pragma unroll
            for (int u = 0; u < 8; u++) x[u] = cluster.map_shared_rank(smv, u)[sidx_row(col)];
        }
        compute(std::integral_constant<int, 3>{}, 1, 0, 3, 0, 0, zero_base);
        typename ST::Pre pre[EPT];
        const auto sctx = st_ctx(st, ptr, t, pr, pidx);
#pragma unroll
        for (int u = 0; u < 8; u++) pre[u] = st_pre(st, sctx, t, (long long)col + ((long long)u << LOGC), pr, pidx);
#pragma unroll
        for (int u = 0; u < 8; u++)
            st_fin(st, sctx, ptr, t, (long long)col + ((long long)u << LOGC), final_value(x[u]), pre[u], pr, pidx);
        if (!async_x) cluster.sync();  // peers keep their shared memory until every gather has finished
    }
}

template <bool INV, int LOGC, class LD, class ST>
__global__ void __launch_bounds__((1 << LOGC) / 8, 65536 / (((1 << LOGC) / 8) * kCapRegs)) ntt_cl8(NttBatch b, int logN, DevPrimes pr, const ulonglong2 *__restrict__ tw,
                                                           const double *__restrict__ twd,
                                                           const NttConst *__restrict__ ncs, LD ld, ST st, bool async_x) {
    extern __shared__ uint64_t sm[];
    __shared__ __align__(8) uint64_t xbar;
    const int t = blockIdx.x >> 3;
    pdl_wait();
    pdl_trigger();
    uint64_t *ptr;
    int pidx;
    if (!locate(b, t, 1 << logN, ptr, pidx)) return;  // uniform over the cluster (same transform)
    if (async_x && threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cl_smem_u32(&xbar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    const NttConst nc = ncs[pidx];
    if (nc.f64) ntt_cl8_body<INV, LOGC, true>(logN, pr, tw, twd, nc, ptr, t, pidx, ld, st, sm, &xbar, async_x);
    else ntt_cl8_body<INV, LOGC, false>(logN, pr, tw, twd, nc, ptr, t, pidx, ld, st, sm, &xbar, async_x);
}

template <bool INV, int LOGC, class LD, class ST>
void launch_cl8(Ctx &c, const NttBatch &b, const LD &ld, const ST &st) {
    constexpr int C = 1 << LOGC;
    const size_t smem = (size_t)C * sizeof(uint64_t) * (INV && cl_st_async() ? 2 : 1);  // inverse: + receive buffer
    auto kern = ntt_cl8<INV, LOGC, LD, ST>;
    ensure_smem(c, (const void *)kern, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)b.count * 8);
    cfg.blockDim = dim3(C / 8);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[3];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 8;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = add_priority_attr(attr, pdl_enabled() ? 2 : 1);
    VR_CUDA(cudaLaunchKernelEx(&cfg, kern, b, c.log_n, c.primes, (const ulonglong2 *)(INV ? c.itw2 : c.tw2),
                               (const double *)(INV ? c.itwd : c.twd), (const NttConst *)c.ntt_const, ld, st, cl_st_async()));
    check_launch("ntt_cl8");
}

// Policy (measured on B200, tools/cl_probe.sh, tools/ab_cl.sh): the cluster kernel beats the two
// passes from ~24 transforms at N <= 2^14 (0.243 -> 0.226 us per 2^14 transform at 1280 transforms;
// cfg 3 +1.5% with the threshold at 24-32 instead of 256).  At 24 the 30-transform ModUp NTT of a
// single relinearisation runs as one cluster kernel: alone the chain is 2.5 us slower, but inside
// matmul_outer (next to the streaming (d0, d1) pass) the step is 1.8% faster (83.6 -> 82.2 us).
// Below ~16 transforms the two passes win (chain 44.7 -> 51.9 us at 8); at N = 2^15 the cluster
// kernel does not pay (512-thread CTAs at 80 registers: one CTA per SM).  VR_NTT_CL = minimum
// batch (default 24; 0 disables).
inline int ntt_cl_min() {
    static const int v = [] {
        const char *e = getenv("VR_NTT_CL");
        return e ? atoi(e) : 24;
    }();
    return v;
}

template <bool INV, class LD, class ST>
bool try_cl8(Ctx &c, const NttBatch &b, const LD &ld, const ST &st, bool force = false) {
    const int lim = ntt_cl_min();
    if (lim <= 0) return false;  // VR_NTT_CL=0 is a kill switch, also for forced callers
    // Inside a slot graph recorded for resident operands (asynchronous matmul_outer, Ctx::capture_cl)
    // every transform is ONE cluster kernel whatever its batch: the overlapped chains are bound by the
    // rate at which the GPU dispatches their small kernels (8 slots: 20 us per 10-kernel chain, 16 us per
    // 7-kernel chain), not by a single chain's latency, which is what the two-pass form wins below ~16
    // transforms (cfg-2 step 43.4 -> 39.6 us per product).
    if (!force && b.count < lim && !(c.capturing && c.capture_cl)) return false;
    switch (c.log_n) {
        case 12: launch_cl8<INV, 9>(c, b, ld, st); return true;
        case 13: launch_cl8<INV, 10>(c, b, ld, st); return true;
        case 14: launch_cl8<INV, 11>(c, b, ld, st); return true;
        default: return false;
    }
}

template <bool INV, class LD, class ST>
void run_fused(Ctx &c, const NttBatch &b, const LD &ld, const ST &st) {
    if (b.count <= 0) return;
    if (try_cl8<INV>(c, b, ld, st)) return;
    const int logN = c.log_n;
    if (c.n <= 4) {
        ntt_tiny<INV><<<nblocks(b.count, 64), 64, 0, c.stream>>>(b, logN, c.primes, INV ? c.itw2 : c.tw2, c.ntt_const, ld, st);
        check_launch("ntt_tiny");
        return;
    }
    if (c.n < 2048) {
        PassArgs a{logN, 0, 1, 1, 0, 0};
        dispatch_pass<INV, false>(c, b, a, logN, 3, ld, st);
        return;
    }
    const int la = logN / 2, lb = logN - la;
    const int T1 = 1 << la, T2 = 1 << lb;
    // small batches are latency-bound: 4 elements per thread halves each thread's chain
    static int small_batch = [] {
        const char *e = getenv("VR_NTT_SMALL");
        return e ? atoi(e) : 64;
    }();
    // (the threshold is in elements: 64 transforms of 2^14; at N = 2^15 a 64-transform batch -- the
    // fused relinearise+rescale of config 5a's four row blocks -- already fills the machine)
    const int le = (long long)b.count * c.n <= (long long)small_batch << 14 ? 2 : 3;
    PassArgs p1{logN, 0, pick_tpc(b.count, 1 << lb, T1, 16, 4, le), 0, 0, 0, le == 2};
    PassArgs p2{logN, la, pick_tpc(b.count, 1 << la, T2, 2048 / T2, 1, le), 0, 0, 0, le == 2};
    // the first pass hands its intermediate to the second (raw doubles on the FP64 body)
    (INV ? p2 : p1).raw_out = 1;
    (INV ? p1 : p2).raw_in = 1;
    if (!INV) {
        p2.last = 1;
        dispatch_pass<false, true>(c, b, p1, la, le, ld, StPlain{});
        dispatch_pass<false, false>(c, b, p2, lb, le, LdPlain{}, st);
    } else {
        p1.last = 1;
        dispatch_pass<true, false>(c, b, p2, lb, le, ld, StPlain{});
        dispatch_pass<true, true>(c, b, p1, la, le, LdPlain{}, st);
    }
}

}  // namespace nttk

template <class LD, class ST>
void ntt_forward_fused(Ctx &c, const NttBatch &b, const LD &ld, const ST &st) { nttk::run_fused<false>(c, b, ld, st); }
template <class LD, class ST>
void ntt_inverse_fused(Ctx &c, const NttBatch &b, const LD &ld, const ST &st) { nttk::run_fused<true>(c, b, ld, st); }
// one-kernel cluster transform regardless of the batch threshold (N <= 2^14; else the two passes)
template <class LD, class ST>
void ntt_inverse_cl(Ctx &c, const NttBatch &b, const LD &ld, const ST &st) {
    if (b.count > 0 && !nttk::try_cl8<true>(c, b, ld, st, true)) nttk::run_fused<true>(c, b, ld, st);
}

}  // namespace vr
