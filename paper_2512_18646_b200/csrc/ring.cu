// ring.cu -- RNS elementwise kernels (add/sub/tensor/plain & scalar products,
// Galois permutation, level drop) and the fused column-ciphertext tensor-sum
// that realises matmul_outer's hot loop (multicipher.py:100-102).
//
// All kernels are HBM-bound streaming passes over [poly][limb][N] uint64
// arrays; each thread handles two adjacent coefficients with 128-bit loads so
// a warp moves 512 contiguous bytes per access.
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdlib>

#include "ring.cuh"
#include "ntt_impl.cuh"

namespace vr {

namespace {

__device__ __forceinline__ ulonglong2 ld2(const uint64_t *p) { return *reinterpret_cast<const ulonglong2 *>(p); }
__device__ __forceinline__ void st2(uint64_t *p, uint64_t a, uint64_t b) {
    *reinterpret_cast<ulonglong2 *>(p) = make_ulonglong2(a, b);
}

// element-pair index -> (ct, poly, limb, k)
struct Idx {
    long long ct;
    int poly, limb, k;
};
__device__ __forceinline__ bool decompose(long long pair, int polys, int nl, int N, Idx &o) {
    const int halfN = N >> 1;
    long long rest = pair / halfN;
    o.k = (int)(pair - rest * halfN) * 2;
    o.limb = (int)(rest % nl);
    rest /= nl;
    o.poly = (int)(rest % polys);
    o.ct = rest / polys;
    return true;
}

__global__ void k_binop(const uint64_t *const *A, const uint64_t *const *B, uint64_t *const *O, int count, int polys,
                        int nl, int N, int op, DevPrimes pr) {
    pdl_wait();
    pdl_trigger();
    const long long pair = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (pair >= (long long)count * polys * nl * (N / 2)) return;
    Idx x;
    decompose(pair, polys, nl, N, x);
    const uint64_t q = pr.m[x.limb].q;
    const size_t off = ((size_t)x.poly * nl + x.limb) * N + x.k;
    ulonglong2 a = ld2(A[x.ct] + off), b = ld2(B[x.ct] + off);
    uint64_t r0, r1;
    if (op == 0) { r0 = add_mod(a.x, b.x, q); r1 = add_mod(a.y, b.y, q); }
    else { r0 = sub_mod(a.x, b.x, q); r1 = sub_mod(a.y, b.y, q); }
    st2(O[x.ct] + off, r0, r1);
}

__global__ void k_tensor(const uint64_t *const *A, const uint64_t *const *B, uint64_t *const *O, int count, int nl, int N,
                         DevPrimes pr) {
    pdl_wait();
    pdl_trigger();
    const long long pair = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (pair >= (long long)count * nl * (N / 2)) return;
    Idx x;
    decompose(pair, 1, nl, N, x);
    const Modulus m = pr.m[x.limb];
    const size_t o0 = (size_t)x.limb * N + x.k, o1 = (size_t)(nl + x.limb) * N + x.k, o2 = (size_t)(2 * nl + x.limb) * N + x.k;
    const uint64_t *a = A[x.ct], *b = B[x.ct];
    uint64_t *d = O[x.ct];
    ulonglong2 a0 = ld2(a + o0), a1 = ld2(a + o1), b0 = ld2(b + o0), b1 = ld2(b + o1);
    st2(d + o0, mul_mod(a0.x, b0.x, m), mul_mod(a0.y, b0.y, m));
    u128 s = mul_wide(a0.x, b1.x), t = mul_wide(a0.y, b1.y);
    mac_to(s, a1.x, b0.x);
    mac_to(t, a1.y, b0.y);
    st2(d + o1, reduce128(s, m), reduce128(t, m));
    st2(d + o2, mul_mod(a1.x, b1.x, m), mul_mod(a1.y, b1.y, m));
}

// out[ct][p][i] = ct[p][i] * pt[ct or shared][i]
__global__ void k_mul_plain(const uint64_t *const *C, const uint64_t *const *P, uint64_t *const *O, int count, int polys,
                            int nl, int N, int shared_pt, DevPrimes pr) {
    pdl_wait();
    pdl_trigger();
    const long long pair = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (pair >= (long long)count * polys * nl * (N / 2)) return;
    Idx x;
    decompose(pair, polys, nl, N, x);
    const Modulus m = pr.m[x.limb];
    const size_t off = ((size_t)x.poly * nl + x.limb) * N + x.k;
    ulonglong2 a = ld2(C[x.ct] + off), b = ld2(P[shared_pt ? 0 : x.ct] + (size_t)x.limb * N + x.k);
    st2(O[x.ct] + off, mul_mod(a.x, b.x, m), mul_mod(a.y, b.y, m));
}

__global__ void k_mul_scalar(const uint64_t *const *C, uint64_t *const *O, int count, int polys, int nl, int N,
                             LimbScalars s, DevPrimes pr) {
    pdl_wait();
    pdl_trigger();
    const long long pair = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (pair >= (long long)count * polys * nl * (N / 2)) return;
    Idx x;
    decompose(pair, polys, nl, N, x);
    const uint64_t q = pr.m[x.limb].q, w = s.v[x.limb], wsh = s.sh[x.limb];
    const size_t off = ((size_t)x.poly * nl + x.limb) * N + x.k;
    ulonglong2 a = ld2(C[x.ct] + off);
    st2(O[x.ct] + off, mul_shoup(a.x, w, wsh, q), mul_shoup(a.y, w, wsh, q));
}

// O[c][p][i] += B[c][p][i] * s_i  where B has nlb >= nl limbs per poly (level-dropped read)
__global__ void k_axpy(uint64_t *const *O, const uint64_t *const *B, int count, int polys, int nl, int nlb, int N,
                       LimbScalars s, DevPrimes pr) {
    pdl_wait();
    pdl_trigger();
    const long long pair = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (pair >= (long long)count * polys * nl * (N / 2)) return;
    Idx x;
    decompose(pair, polys, nl, N, x);
    const uint64_t q = pr.m[x.limb].q, w = s.v[x.limb], wsh = s.sh[x.limb];
    uint64_t *o = O[x.ct] + ((size_t)x.poly * nl + x.limb) * N + x.k;
    const ulonglong2 b = ld2(B[x.ct] + ((size_t)x.poly * nlb + x.limb) * N + x.k);
    const ulonglong2 a = ld2(o);
    st2(o, add_mod(a.x, mul_shoup(b.x, w, wsh, q), q), add_mod(a.y, mul_shoup(b.y, w, wsh, q), q));
}

// O[c][p][i] = C[c][p][i] * s_i + B[c][p][i] * t_i  (B with nlb >= nl limbs): mul_scalar + axpy in one pass
__global__ void k_scale_axpy(const uint64_t *const *C, const uint64_t *const *B, uint64_t *const *O, int count, int polys,
                             int nl, int nlb, int N, LimbScalars s, LimbScalars t, DevPrimes pr) {
    pdl_wait();
    pdl_trigger();
    const long long pair = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (pair >= (long long)count * polys * nl * (N / 2)) return;
    Idx x;
    decompose(pair, polys, nl, N, x);
    const uint64_t q = pr.m[x.limb].q, w = s.v[x.limb], wsh = s.sh[x.limb], u = t.v[x.limb], ush = t.sh[x.limb];
    const size_t off = ((size_t)x.poly * nl + x.limb) * N + x.k;
    const ulonglong2 a = ld2(C[x.ct] + off), b = ld2(B[x.ct] + ((size_t)x.poly * nlb + x.limb) * N + x.k);
    st2(O[x.ct] + off, add_mod(mul_shoup(a.x, w, wsh, q), mul_shoup(b.x, u, ush, q), q),
        add_mod(mul_shoup(a.y, w, wsh, q), mul_shoup(b.y, u, ush, q), q));
}

__global__ void k_add_const(uint64_t *const *C, int count, int nl, int N, LimbScalars s, DevPrimes pr) {
    pdl_wait();
    pdl_trigger();
    const long long pair = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (pair >= (long long)count * nl * (N / 2)) return;
    Idx x;
    decompose(pair, 1, nl, N, x);
    const uint64_t q = pr.m[x.limb].q, v = s.v[x.limb];
    uint64_t *p = C[x.ct] + (size_t)x.limb * N + x.k;
    ulonglong2 a = ld2(p);
    st2(p, add_mod(a.x, v, q), add_mod(a.y, v, q));
}

// out[k] = in[perm_g(k)],  perm_g(k) = br(((2 br(k) + 1) g mod 2N - 1) / 2)
__device__ __forceinline__ int galois_src(int k, uint32_t g, int logN) {
    const uint32_t brk = __brev((uint32_t)k) >> (32 - logN);
    const uint32_t e = ((2u * brk + 1u) * g) & ((2u << logN) - 1u);
    return (int)(__brev((e - 1u) >> 1) >> (32 - logN));
}

__global__ void k_permute(const uint64_t *const *C, uint64_t *const *O, int count, int polys, int nl, int logN, uint32_t g) {
    pdl_wait();
    pdl_trigger();
    const int N = 1 << logN;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)count * polys * nl * N) return;
    const int k = (int)(e & (N - 1));
    const long long row = e >> logN;  // (ct, poly, limb)
    const long long ct = row / ((long long)polys * nl);
    const size_t roff = (size_t)(row - ct * polys * nl) * N;
    O[ct][roff + k] = C[ct][roff + galois_src(k, g, logN)];
}

__global__ void k_copy_limbs(const uint64_t *const *C, uint64_t *const *O, int count, int polys, int nl_in, int nl_out,
                             int limb0, int N) {
    pdl_wait();
    pdl_trigger();
    const long long pair = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (pair >= (long long)count * polys * nl_out * (N / 2)) return;
    Idx x;
    decompose(pair, polys, nl_out, N, x);
    ulonglong2 a = ld2(C[x.ct] + ((size_t)x.poly * nl_in + x.limb + limb0) * N + x.k);
    st2(O[x.ct] + ((size_t)x.poly * nl_out + x.limb) * N + x.k, a.x, a.y);
}

__global__ void k_mod_fixup(uint64_t *data, long long count_polys, int nl, int N, DevPrimes pr) {
    pdl_wait();
    pdl_trigger();
    const long long pair = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (pair >= count_polys * nl * (N / 2)) return;
    Idx x;
    decompose(pair, 1, nl, N, x);
    const Modulus m = pr.m[x.limb];
    uint64_t *p = data + ((size_t)x.ct * nl + x.limb) * N + x.k;
    ulonglong2 a = ld2(p);
    st2(p, reduce64(a.x, m), reduce64(a.y, m));
}

// ---- TMA bulk-copy + mbarrier helpers (sm_90+/sm_100a PTX) ----------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done)
                     : "r"(smem_u32(bar)), "r"(parity)
                     : "memory");
    } while (!done);
}
// global -> shared bulk copy (TMA engine, no tensor map), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// same, with an L2 eviction-priority policy (createpolicy) attached to the transfer
__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
                     "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// Fused sum_k tensor(L[b][k], R[k]) for NB row blocks sharing the right operand.
// Grid (coefficient tiles of TS_TILE, limbs, TS_SPLIT): the TS_SPLIT CTAs of a
// thread-block cluster take disjoint parts of the k range.  Inside a CTA one
// producer warp streams the 2*NB + 2 limb tiles of every k into an
// TS_STAGES-deep shared-memory ring with TMA bulk copies (cp.async.bulk +
// mbarrier expect_tx), so ~64 KB per CTA are always in flight; the consumer
// warps accumulate the 64x64 -> 128-bit products (folded mod q every 8 terms).
// Partials are reduced mod q and combined through distributed shared memory;
// cluster rank 0 writes the degree-2 result.  R is streamed once per group.
template <int NB, int TILE, int MAXST = 8>
__host__ __device__ constexpr int ts_stages() {
    // ring of (2 NB + 2) limb tiles per stage, <= ~200 KB of shared memory, 2..8 stages
    return (200 * 1024) / ((2 * NB + 2) * TILE * 8) > MAXST ? MAXST
           : ((200 * 1024) / ((2 * NB + 2) * TILE * 8) < 2 ? 2 : (200 * 1024) / ((2 * NB + 2) * TILE * 8));
}

// MODE 0: (d0, d1, d2); MODE 1: d2 = sum L1 R1 only (reads half the operands); MODE 2: (d0, d1) only.
template <int NB, int TS_TILE, int TS_SPLIT, int MAXST, int MODE>
__global__ void __launch_bounds__(TS_TILE / 2 + 32)
    k_tensor_sum(const uint64_t *const *L, const uint64_t *const *R, int n, int nl, int N, DevPrimes pr, uint64_t *const *O,
                 int hint, int rb) {
    pdl_wait();
    pdl_trigger();
    // rb > 1: rb independent row blocks interleaved along x (block fastest), so the rb CTAs that read
    // the same R tiles are dispatched together and share them through L2
    const int xb = rb > 1 ? (int)blockIdx.x % rb : 0;
    const int xt = rb > 1 ? (int)blockIdx.x / rb : (int)blockIdx.x;
    L += (size_t)xb * NB * n;
    O += xb * NB;
    constexpr int TS_CONSUMERS = TS_TILE / 2;  // 2 coefficients per consumer thread
    constexpr int TS_STAGES = ts_stages<NB, TS_TILE, MAXST>();
    // limb tiles per stage: L[b] poly0/poly1 ..., R poly0/poly1 (MODE 1: L[b] poly1 ..., R poly1)
    constexpr int ARR = MODE == 1 ? NB + 1 : 2 * NB + 2;
    constexpr int P0 = MODE == 1 ? 2 : 0, P1 = MODE == 2 ? 2 : 3;  // output polys [P0, P1)
    extern __shared__ __align__(128) uint64_t ts_smem[];
    uint64_t *ring = ts_smem;                                        // [STAGES][ARR][tile]
    __shared__ __align__(8) uint64_t full[TS_STAGES], empty[TS_STAGES];
    // partials reuse the ring after the stream is drained: [NB*3][TS_CONSUMERS]
    ulonglong2(*part)[TS_CONSUMERS] = reinterpret_cast<ulonglong2(*)[TS_CONSUMERS]>(ts_smem);
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int tile = N < TS_TILE ? N : TS_TILE;
    const int cons = tile / 2;
    const int k0 = xt * tile, i = blockIdx.y;
    const int z = (int)cluster.block_rank();
    const int per = (n + TS_SPLIT - 1) / TS_SPLIT;
    const int tb = min(n, z * per), te = min(n, tb + per);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int producer_warp = TS_CONSUMERS / 32;  // the last warp
    const int nwarps_cons = (cons + 31) / 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < TS_STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], nwarps_cons);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const Modulus m = pr.m[i];
    if (warp == producer_warp) {
        if (lane == 0) {
            const uint64_t pol_keep = policy_evict_last(), pol_drop = policy_evict_first();
            (void)pol_keep;
            (void)pol_drop;
            const uint32_t bytes = (uint32_t)tile * 8;
            const size_t o0 = (size_t)i * N + k0, o1 = (size_t)(nl + i) * N + k0;
            for (int t = tb, it = 0; t < te; t++, it++) {
                const int s = it % TS_STAGES;
                if (it >= TS_STAGES) mbar_wait(&empty[s], ((it / TS_STAGES) - 1) & 1);
                uint64_t *st = ring + (size_t)s * ARR * tile;
                mbar_expect_tx(&full[s], bytes * ARR);
                if constexpr (MODE == 1) {
                    // hint bit 0: keep the c1 halves in L2 for the (d0, d1) pass that follows
                    if (hint & 1) {
#pragma unroll
                        for (int b = 0; b < NB; b++) bulk_g2s_hint(st + b * tile, L[b * n + t] + o1, bytes, &full[s], pol_keep);
                        bulk_g2s_hint(st + NB * tile, R[t] + o1, bytes, &full[s], pol_keep);
                    } else {
#pragma unroll
                        for (int b = 0; b < NB; b++) bulk_g2s(st + b * tile, L[b * n + t] + o1, bytes, &full[s]);
                        bulk_g2s(st + NB * tile, R[t] + o1, bytes, &full[s]);
                    }
                } else if (MODE == 2 && hint) {
                    // last use of every operand: stream them through L2 at the lowest priority
#pragma unroll
                    for (int b = 0; b < NB; b++) {
                        const uint64_t *l = L[b * n + t];
                        bulk_g2s_hint(st + (2 * b) * tile, l + o0, bytes, &full[s], pol_drop);
                        bulk_g2s_hint(st + (2 * b + 1) * tile, l + o1, bytes, &full[s], pol_drop);
                    }
                    const uint64_t *r = R[t];
                    bulk_g2s_hint(st + (2 * NB) * tile, r + o0, bytes, &full[s], pol_drop);
                    bulk_g2s_hint(st + (2 * NB + 1) * tile, r + o1, bytes, &full[s], pol_drop);
                } else {
#pragma unroll
                    for (int b = 0; b < NB; b++) {
                        const uint64_t *l = L[b * n + t];
                        bulk_g2s(st + (2 * b) * tile, l + o0, bytes, &full[s]);
                        bulk_g2s(st + (2 * b + 1) * tile, l + o1, bytes, &full[s]);
                    }
                    const uint64_t *r = R[t];
                    bulk_g2s(st + (2 * NB) * tile, r + o0, bytes, &full[s]);
                    bulk_g2s(st + (2 * NB + 1) * tile, r + o1, bytes, &full[s]);
                }
            }
        }
    }
    u128 acc[NB][3][2];
    if (warp != producer_warp && threadIdx.x < cons) {
#pragma unroll
        for (int b = 0; b < NB; b++)
#pragma unroll
            for (int p = 0; p < 3; p++)
#pragma unroll
                for (int e = 0; e < 2; e++) acc[b][p][e] = u128{0, 0};
        const int c2 = threadIdx.x * 2;
        const int live = cons - warp * 32;  // consumer lanes in this warp (small N: partial warp)
        const unsigned wmask = live >= 32 ? 0xffffffffu : ((1u << live) - 1u);
        for (int t = tb, it = 0; t < te; t++, it++) {
            const int s = it % TS_STAGES;
            mbar_wait(&full[s], (it / TS_STAGES) & 1);
            const uint64_t *st = ring + (size_t)s * ARR * tile;
            if (hint & 8) {  // diagnostic (VR_TS_HINT bit 3): stream only, no arithmetic
                __syncwarp(wmask);
                if (lane == 0) mbar_arrive(&empty[s]);
                continue;
            }
            // copy this thread's operands out of the slot and release it BEFORE the arithmetic, so
            // the producer refills it while the products run (one more stage of effective buffering)
            ulonglong2 r0, r1, l0[NB], l1[NB];
            if constexpr (MODE == 1) {
                r1 = *reinterpret_cast<const ulonglong2 *>(st + NB * tile + c2);
#pragma unroll
                for (int b = 0; b < NB; b++) l1[b] = *reinterpret_cast<const ulonglong2 *>(st + b * tile + c2);
            } else {
                r0 = *reinterpret_cast<const ulonglong2 *>(st + (2 * NB) * tile + c2);
                r1 = *reinterpret_cast<const ulonglong2 *>(st + (2 * NB + 1) * tile + c2);
#pragma unroll
                for (int b = 0; b < NB; b++) {
                    l0[b] = *reinterpret_cast<const ulonglong2 *>(st + (2 * b) * tile + c2);
                    l1[b] = *reinterpret_cast<const ulonglong2 *>(st + (2 * b + 1) * tile + c2);
                }
            }
            __syncwarp(wmask);
            if (lane == 0) mbar_arrive(&empty[s]);
            if constexpr (MODE == 1) {
#pragma unroll
                for (int b = 0; b < NB; b++) {
                    mac_to(acc[b][2][0], l1[b].x, r1.x);
                    mac_to(acc[b][2][1], l1[b].y, r1.y);
                }
            } else {
#pragma unroll
                for (int b = 0; b < NB; b++) {
                    mac_to(acc[b][0][0], l0[b].x, r0.x);
                    mac_to(acc[b][0][1], l0[b].y, r0.y);
                    if constexpr (MODE == 0) {
                        // Karatsuba: three 64x64 products instead of four.  acc[1] collects
                        // (l0 + l1)(r0 + r1) (< 2^124: residues < 2^61); d1 = that - d0 - d2 at the end.
                        mac_to(acc[b][2][0], l1[b].x, r1.x);
                        mac_to(acc[b][2][1], l1[b].y, r1.y);
                        mac_to(acc[b][1][0], l0[b].x + l1[b].x, r0.x + r1.x);
                        mac_to(acc[b][1][1], l0[b].y + l1[b].y, r0.y + r1.y);
                    } else {
                        mac_to(acc[b][1][0], l0[b].x, r1.x);
                        mac_to(acc[b][1][1], l0[b].y, r1.y);
                        mac_to(acc[b][1][0], l1[b].x, r0.x);
                        mac_to(acc[b][1][1], l1[b].y, r0.y);
                    }
                }
            }
            if ((it & 7) == 7) {
#pragma unroll
                for (int b = 0; b < NB; b++)
#pragma unroll
                    for (int p = P0; p < P1; p++)
#pragma unroll
                        for (int e = 0; e < 2; e++) acc[b][p][e] = u128{reduce128(acc[b][p][e], m), 0};
            }
        }
    }
    __syncthreads();  // ring drained: reuse it for the partials
    if (warp != producer_warp && threadIdx.x < cons) {
#pragma unroll
        for (int b = 0; b < NB; b++) {
            uint64_t v[3][2];
#pragma unroll
            for (int p = P0; p < P1; p++)
#pragma unroll
                for (int e = 0; e < 2; e++) v[p][e] = reduce128(acc[b][p][e], m);
            if constexpr (MODE == 0) {  // undo Karatsuba: d1 = (l0 + l1)(r0 + r1) - d0 - d2
#pragma unroll
                for (int e = 0; e < 2; e++) v[1][e] = sub_mod(sub_mod(v[1][e], v[0][e], m.q), v[2][e], m.q);
            }
#pragma unroll
            for (int p = P0; p < P1; p++) part[b * 3 + p][threadIdx.x] = make_ulonglong2(v[p][0], v[p][1]);
        }
    }
    cluster.sync();
    if (z == 0 && threadIdx.x < cons) {
        const int k = k0 + threadIdx.x * 2;
#pragma unroll
        for (int b = 0; b < NB; b++) {
            uint64_t *o = O[b];
#pragma unroll
            for (int p = P0; p < P1; p++) {
                ulonglong2 v = part[b * 3 + p][threadIdx.x];
#pragma unroll
                for (int r = 1; r < TS_SPLIT; r++) {
                    const ulonglong2 w = cluster.map_shared_rank(&part[b * 3 + p][0], r)[threadIdx.x];
                    v.x = add_mod(v.x, w.x, m.q);
                    v.y = add_mod(v.y, w.y, m.q);
                }
                st2(o + (size_t)(p * nl + i) * N + k, v.x, v.y);
            }
        }
    }
    cluster.sync();  // peers keep their shared memory alive until rank 0 has read it
}

// ---- cluster-multicast tensor sum: NB row blocks sharing R, R read from HBM once ---------------
// multicast variant of bulk_g2s: the tile lands at the same shared-memory offset in every CTA of
// `mask` and signals the mbarrier at the same offset in each of them
__device__ __forceinline__ void bulk_g2s_mc(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
        : "memory");
}
// arrive on the barrier at the same offset in cluster CTA `cta` (release at cluster scope)
__device__ __forceinline__ void mbar_arrive_remote(uint64_t *bar, uint32_t cta) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(bar)), "r"(cta));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

// (d0, d1, d2)[b] = sum_k L[b][k] (x) R[k] for NB row blocks (config 5a: 4 blocks of 64 x 256 column
// ciphertexts sharing the 256 right ciphertexts).  One thread-block cluster = NB x SPLIT CTAs: CTA
// (b, z) accumulates row block b over the z-th part of the k range, so each CTA holds one block's
// 128-bit accumulators (no register pressure from NB).  Each CTA's producer thread streams its own
// L_b limb tiles with TMA bulk copies; the R tiles of step k are fetched ONCE per split group by one
// CTA (rotating with k) and multicast into all NB CTAs' rings.  A ring slot is reused only after the
// consumers of all NB CTAs released it (remote mbarrier arrivals), so R crosses HBM once instead of
// once per row block: 5.4 GB instead of 6.4 GB per config-5a product.
template <int NB, int TILE, int SPLIT, int ST>
__global__ void __launch_bounds__(TILE / 2 + 32)
    k_tensor_sum_mc(const uint64_t *const *L, const uint64_t *const *R, int n, int nl, int N, DevPrimes pr, uint64_t *const *O) {
    pdl_wait();
    pdl_trigger();
    constexpr int CONS = TILE / 2;  // 2 coefficients per consumer thread
    constexpr int NWC = CONS / 32;  // consumer warps; the producer warp follows them
    extern __shared__ __align__(128) uint64_t ts_smem[];
    uint64_t *ring = ts_smem;  // [ST][4][TILE]: L poly 0, L poly 1, R poly 0, R poly 1
    __shared__ __align__(8) uint64_t full[ST], empty[ST];
    ulonglong2(*part)[CONS] = reinterpret_cast<ulonglong2(*)[CONS]>(ts_smem);  // [3][CONS] after the stream
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int b = rank % NB, zk = rank / NB;
    const int k0 = blockIdx.x * TILE, i = blockIdx.y;
    const int per = (n + SPLIT - 1) / SPLIT;
    const int tb = min(n, zk * per), te = min(n, tb + per);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint16_t mask = (uint16_t)(((1u << NB) - 1u) << (zk * NB));
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NWC * NB);  // every consumer warp of the NB CTAs of this split group
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster.sync();  // barriers initialised cluster-wide before any multicast or remote arrival
    const Modulus m = pr.m[i];
    if (warp == NWC) {
        if (lane == 0) {
            const uint32_t bytes = (uint32_t)TILE * 8;
            const size_t o0 = (size_t)i * N + k0, o1 = (size_t)(nl + i) * N + k0;
            for (int t = tb, it = 0; t < te; t++, it++) {
                const int s = it % ST;
                if (it >= ST) mbar_wait_cluster(&empty[s], ((it / ST) - 1) & 1);
                uint64_t *st = ring + (size_t)s * 4 * TILE;
                mbar_expect_tx(&full[s], bytes * 4);
                const uint64_t *l = L[(size_t)b * n + t];
                bulk_g2s(st, l + o0, bytes, &full[s]);
                bulk_g2s(st + TILE, l + o1, bytes, &full[s]);
                if (it % NB == b) {
                    const uint64_t *r = R[t];
                    bulk_g2s_mc(st + 2 * TILE, r + o0, bytes, &full[s], mask);
                    bulk_g2s_mc(st + 3 * TILE, r + o1, bytes, &full[s], mask);
                }
            }
        }
    } else {
        u128 acc[3][2];
#pragma unroll
        for (int p = 0; p < 3; p++) acc[p][0] = acc[p][1] = u128{0, 0};
        const int c2 = threadIdx.x * 2;
        for (int t = tb, it = 0; t < te; t++, it++) {
            const int s = it % ST;
            mbar_wait(&full[s], (it / ST) & 1);
            const uint64_t *st = ring + (size_t)s * 4 * TILE;
            const ulonglong2 l0 = *reinterpret_cast<const ulonglong2 *>(st + c2);
            const ulonglong2 l1 = *reinterpret_cast<const ulonglong2 *>(st + TILE + c2);
            const ulonglong2 r0 = *reinterpret_cast<const ulonglong2 *>(st + 2 * TILE + c2);
            const ulonglong2 r1 = *reinterpret_cast<const ulonglong2 *>(st + 3 * TILE + c2);
            mac_to(acc[0][0], l0.x, r0.x);
            mac_to(acc[0][1], l0.y, r0.y);
            mac_to(acc[1][0], l0.x, r1.x);
            mac_to(acc[1][1], l0.y, r1.y);
            mac_to(acc[1][0], l1.x, r0.x);
            mac_to(acc[1][1], l1.y, r0.y);
            mac_to(acc[2][0], l1.x, r1.x);
            mac_to(acc[2][1], l1.y, r1.y);
            __syncwarp();
            if (lane < NB) mbar_arrive_remote(&empty[s], (uint32_t)(zk * NB + lane));  // release slot s in all NB CTAs
            if ((it & 7) == 7) {
#pragma unroll
                for (int p = 0; p < 3; p++)
#pragma unroll
                    for (int e = 0; e < 2; e++) acc[p][e] = u128{reduce128(acc[p][e], m), 0};
            }
        }
        __syncwarp();
        // every multicast into this ring has landed (all its steps were consumed): reuse it
        asm volatile("bar.sync 1, %0;" ::"r"(CONS) : "memory");
#pragma unroll
        for (int p = 0; p < 3; p++) part[p][threadIdx.x] = make_ulonglong2(reduce128(acc[p][0], m), reduce128(acc[p][1], m));
    }
    cluster.sync();
    if (zk == 0 && threadIdx.x < CONS) {
        const int k = k0 + threadIdx.x * 2;
        uint64_t *o = O[b];
#pragma unroll
        for (int p = 0; p < 3; p++) {
            ulonglong2 v = part[p][threadIdx.x];
#pragma unroll
            for (int r = 1; r < SPLIT; r++) {
                const ulonglong2 w = cluster.map_shared_rank(&part[p][0], r * NB + b)[threadIdx.x];
                v.x = add_mod(v.x, w.x, m.q);
                v.y = add_mod(v.y, w.y, m.q);
            }
            st2(o + (size_t)(p * nl + i) * N + k, v.x, v.y);
        }
    }
    cluster.sync();  // peers keep their shared memory alive until the group's rank 0 has read it
}

constexpr int TB = 256;

// Integer-pipe roofline probe: the NTT's Harvey/Shoup forward butterfly on registers only,
// 8 independent chains per thread (no memory traffic).  bench.py divides the NTT's achieved
// butterflies/s by this peak.
__global__ void __launch_bounds__(256) k_bfly_peak(uint64_t q, uint64_t w, uint64_t wsh, int iters, uint64_t *sink) {
    uint64_t x[8], y[8];
    const uint64_t q2 = 2 * q;
#pragma unroll
    for (int e = 0; e < 8; e++) {
        x[e] = (threadIdx.x * 977u + e * 131u) % q;
        y[e] = (blockIdx.x * 613u + e * 71u) % q;
    }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int e = 0; e < 8; e++) {
            const uint64_t xx = x[e] >= q2 ? x[e] - q2 : x[e];
            const uint64_t t = mul_shoup_lazy(y[e], w, wsh, q);
            x[e] = xx + t;
            y[e] = xx - t + q2;
        }
    }
    uint64_t acc = 0;
#pragma unroll
    for (int e = 0; e < 8; e++) acc ^= x[e] ^ y[e];
    if (acc == 0x12345) sink[0] = acc;  // keep the chains alive
}

// FP64-pipe peak: the NTT's FP64 butterfly (nttk::mulmod_f, x + t, x - t) on registers only; one fold
// per 8 butterflies keeps |x| bounded (a forward pass folds never, so this peak is conservative).
__global__ void __launch_bounds__(256) k_bfly_peak_f64(double q, double w, double qinv, int iters, double *sink) {
    double x[8], y[8];
#pragma unroll
    for (int e = 0; e < 8; e++) {
        x[e] = (double)((threadIdx.x * 977u + e * 131u) % 1000003u);
        y[e] = (double)((blockIdx.x * 613u + e * 71u) % 1000003u);
    }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int r = 0; r < 8; r++) {
#pragma unroll
            for (int e = 0; e < 8; e++) {
                const double t = nttk::mulmod_f(y[e], w, q, qinv);
                const double a = x[e];
                x[e] = __dadd_rn(a, t);
                y[e] = __dsub_rn(a, t);
            }
        }
#pragma unroll
        for (int e = 0; e < 8; e++) {
            x[e] = nttk::fold_f(x[e], q, qinv);
            y[e] = nttk::fold_f(y[e], q, qinv);
        }
    }
    double acc = 0;
#pragma unroll
    for (int e = 0; e < 8; e++) acc += x[e] + y[e];
    if (acc == 12345.0) sink[0] = acc;
}

}  // namespace

void bfly_peak_f64(Ctx &c, int blocks, int iters, uint64_t *sink) {
    int p = 0;
    while (p + 1 < c.np && c.q[p] >= (1ull << 46)) p++;
    const double q = (double)c.q[p];
    k_bfly_peak_f64<<<blocks, 256, 0, c.stream>>>(q, (double)(1234567 % c.q[p]), 1.0 / q, iters, (double *)sink);
    check_launch("k_bfly_peak_f64");
}

void bfly_peak(Ctx &c, int blocks, int iters, uint64_t *sink) {
    const uint64_t q = c.q[1 < c.np ? 1 : 0];
    const uint64_t w = 1234567 % q, wsh = (uint64_t)(((unsigned __int128)w << 64) / q);
    k_bfly_peak<<<blocks, 256, 0, c.stream>>>(q, w, wsh, iters, sink);
    check_launch("k_bfly_peak");
}

LimbScalars limb_scalars(const Ctx &c, int64_t s, int nl) {
    LimbScalars r;
    for (int i = 0; i < nl; i++) {
        const Modulus &m = c.primes.m[i];
        uint64_t v = from_i64(s, m);
        r.v[i] = v;
        r.sh[i] = (uint64_t)(((unsigned __int128)v << 64) / m.q);
    }
    return r;
}

void binop(Ctx &c, const uint64_t *const *A, const uint64_t *const *B, uint64_t *const *O, int count, int polys, int nl, int op) {
    const long long pairs = (long long)count * polys * nl * (c.n / 2);
    if (!pairs) return;
    launch_pdl(k_binop, dim3(nblocks(pairs, TB)), dim3(TB), 0, c.stream, A, B, O, count, polys, nl, c.n, op, c.primes);
    check_launch("k_binop");
}

void tensor(Ctx &c, const uint64_t *const *A, const uint64_t *const *B, uint64_t *const *O, int count, int nl) {
    const long long pairs = (long long)count * nl * (c.n / 2);
    launch_pdl(k_tensor, dim3(nblocks(pairs, TB)), dim3(TB), 0, c.stream, A, B, O, count, nl, c.n, c.primes);
    check_launch("k_tensor");
}

void mul_plain(Ctx &c, const uint64_t *const *C, const uint64_t *const *P, uint64_t *const *O, int count, int polys, int nl,
               int shared_pt) {
    const long long pairs = (long long)count * polys * nl * (c.n / 2);
    launch_pdl(k_mul_plain, dim3(nblocks(pairs, TB)), dim3(TB), 0, c.stream, C, P, O, count, polys, nl, c.n, shared_pt, c.primes);
    check_launch("k_mul_plain");
}

void mul_scalar(Ctx &c, const uint64_t *const *C, uint64_t *const *O, int count, int polys, int nl, const LimbScalars &s) {
    const long long pairs = (long long)count * polys * nl * (c.n / 2);
    launch_pdl(k_mul_scalar, dim3(nblocks(pairs, TB)), dim3(TB), 0, c.stream, C, O, count, polys, nl, c.n, s, c.primes);
    check_launch("k_mul_scalar");
}

void axpy(Ctx &c, uint64_t *const *O, const uint64_t *const *B, int count, int polys, int nl, int nlb, const LimbScalars &s) {
    const long long pairs = (long long)count * polys * nl * (c.n / 2);
    launch_pdl(k_axpy, dim3(nblocks(pairs, TB)), dim3(TB), 0, c.stream, O, B, count, polys, nl, nlb, c.n, s, c.primes);
    check_launch("k_axpy");
}

void scale_axpy(Ctx &c, const uint64_t *const *C, const uint64_t *const *B, uint64_t *const *O, int count, int polys, int nl,
                int nlb, const LimbScalars &s, const LimbScalars &t) {
    const long long pairs = (long long)count * polys * nl * (c.n / 2);
    launch_pdl(k_scale_axpy, dim3(nblocks(pairs, TB)), dim3(TB), 0, c.stream, C, B, O, count, polys, nl, nlb, c.n, s, t,
               c.primes);
    check_launch("k_scale_axpy");
}

void add_const(Ctx &c, uint64_t *const *C, int count, int nl, const LimbScalars &s) {
    const long long pairs = (long long)count * nl * (c.n / 2);
    launch_pdl(k_add_const, dim3(nblocks(pairs, TB)), dim3(TB), 0, c.stream, C, count, nl, c.n, s, c.primes);
    check_launch("k_add_const");
}

void permute(Ctx &c, const uint64_t *const *C, uint64_t *const *O, int count, int polys, int nl, uint32_t g) {
    const long long el = (long long)count * polys * nl * c.n;
    launch_pdl(k_permute, dim3(nblocks(el, TB)), dim3(TB), 0, c.stream, C, O, count, polys, nl, c.log_n, g);
    check_launch("k_permute");
}

void copy_limbs(Ctx &c, const uint64_t *const *C, uint64_t *const *O, int count, int polys, int nl_in, int nl_out, int limb0) {
    const long long pairs = (long long)count * polys * nl_out * (c.n / 2);
    if (!pairs) return;
    launch_pdl(k_copy_limbs, dim3(nblocks(pairs, TB)), dim3(TB), 0, c.stream, C, O, count, polys, nl_in, nl_out, limb0, c.n);
    check_launch("k_copy_limbs");
}

void mod_fixup(Ctx &c, uint64_t *data, long long count_polys, int nl) {
    const long long pairs = count_polys * nl * (c.n / 2);
    launch_pdl(k_mod_fixup, dim3(nblocks(pairs, TB)), dim3(TB), 0, c.stream, data, count_polys, nl, c.n, c.primes);
    check_launch("k_mod_fixup");
}

// Launch shape (tile, split-K) -- tuned on B200 with tools/bw_probe.py; VR_TS_VARIANT overrides.
template <int NB, int TILE, int SPLIT, int MAXST = 8, int MODE = 0>
static void launch_ts(Ctx &c, const uint64_t *const *L, const uint64_t *const *R, int n, int nl, uint64_t *const *O, int rb = 1) {
    constexpr int ARR = MODE == 1 ? NB + 1 : 2 * NB + 2;
    const int tile = c.n < TILE ? c.n : TILE;
    size_t smem = (size_t)ts_stages<NB, TILE, MAXST>() * ARR * tile * sizeof(uint64_t);
    smem = std::max<size_t>(smem, (size_t)NB * 3 * (TILE / 2) * 16);
    auto kern = k_tensor_sum<NB, TILE, SPLIT, MAXST, MODE>;
    ensure_smem(c, (const void *)kern, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c.n / tile * rb, nl, SPLIT);
    cfg.blockDim = dim3(TILE / 2 + 32, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = SPLIT;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    static const int hint = [] {
        const char *e = getenv("VR_TS_HINT");
        return e ? atoi(e) : 1;
    }();
    VR_CUDA(cudaLaunchKernelEx(&cfg, kern, L, R, n, nl, c.n, c.primes, O, hint, rb));
}

template <int NB, int TILE, int SPLIT, int ST>
static void launch_ts_mc(Ctx &c, const uint64_t *const *L, const uint64_t *const *R, int n, int nl, uint64_t *const *O) {
    const size_t smem = std::max<size_t>((size_t)ST * 4 * TILE * sizeof(uint64_t), (size_t)3 * (TILE / 2) * 16);
    auto kern = k_tensor_sum_mc<NB, TILE, SPLIT, ST>;
    ensure_smem(c, (const void *)kern, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c.n / TILE, nl, NB * SPLIT);
    cfg.blockDim = dim3(TILE / 2 + 32, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = NB * SPLIT;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    VR_CUDA(cudaLaunchKernelEx(&cfg, kern, L, R, n, nl, c.n, c.primes, O));
}

template <int NB>
static void ts_variant(Ctx &c, int v, const uint64_t *const *L, const uint64_t *const *R, int n, int nl, uint64_t *const *O) {
    switch (v) {
        case 1: launch_ts<NB, 256, 1, 8>(c, L, R, n, nl, O); break;
        case 2: launch_ts<NB, 128, 2, 8>(c, L, R, n, nl, O); break;
        case 3: launch_ts<NB, 512, 2, 4>(c, L, R, n, nl, O); break;
        case 4: launch_ts<NB, 512, 4, 4>(c, L, R, n, nl, O); break;
        case 5: launch_ts<NB, 256, 2, 8>(c, L, R, n, nl, O); break;
        case 6: launch_ts<NB, 512, 2, 6>(c, L, R, n, nl, O); break;
        case 7: launch_ts<NB, 1024, 2, 2>(c, L, R, n, nl, O); break;
        case 8: launch_ts<NB, 256, 4, 4>(c, L, R, n, nl, O); break;
        default: launch_ts<NB, 256, 2, 4>(c, L, R, n, nl, O); break;  // best on B200 (tools/bw_probe.py)
    }
}

void tensor_sum_mode(Ctx &c, const uint64_t *const *L, const uint64_t *const *R, int n, int nb, int nl, uint64_t *const *O,
                     int mode) {
    if (nb != 1) throw VrError(3, "split tensor_sum supports one row block");
    static const int v2 = [] {
        const char *e = getenv("VR_TS2_VARIANT");
        return e ? atoi(e) : 0;
    }();
    // launch shapes swept on B200 with tools/ts2_sweep.sh (VR_TS1_VARIANT / VR_TS2_VARIANT override)
    static const int v1 = [] {
        const char *e = getenv("VR_TS1_VARIANT");
        return e ? atoi(e) : 0;
    }();
    if (mode == 1) {
        switch (v1) {
            case 1: launch_ts<1, 512, 2, 8, 1>(c, L, R, n, nl, O); break;
            case 2: launch_ts<1, 512, 2, 4, 1>(c, L, R, n, nl, O); break;
            case 3: launch_ts<1, 1024, 2, 4, 1>(c, L, R, n, nl, O); break;
            case 4: launch_ts<1, 256, 4, 8, 1>(c, L, R, n, nl, O); break;
            case 5: launch_ts<1, 256, 2, 8, 1>(c, L, R, n, nl, O); break;
            case 6: launch_ts<1, 128, 4, 8, 1>(c, L, R, n, nl, O); break;
            case 7: launch_ts<1, 256, 8, 8, 1>(c, L, R, n, nl, O); break;
            default: launch_ts<1, 512, 4, 4, 1>(c, L, R, n, nl, O); break;  // 17.9 us alone (was 20.5)
        }
    } else {
        switch (v2) {
            case 1: launch_ts<1, 256, 1, 4, 2>(c, L, R, n, nl, O); break;
            case 2: launch_ts<1, 256, 2, 8, 2>(c, L, R, n, nl, O); break;
            case 3: launch_ts<1, 256, 2, 4, 2>(c, L, R, n, nl, O); break;
            case 4: launch_ts<1, 128, 2, 8, 2>(c, L, R, n, nl, O); break;
            case 5: launch_ts<1, 256, 4, 4, 2>(c, L, R, n, nl, O); break;
            case 6: launch_ts<1, 512, 1, 4, 2>(c, L, R, n, nl, O); break;
            case 7: launch_ts<1, 1024, 2, 2, 2>(c, L, R, n, nl, O); break;
            case 8: launch_ts<1, 512, 2, 6, 2>(c, L, R, n, nl, O); break;
            case 9: launch_ts<1, 512, 4, 4, 2>(c, L, R, n, nl, O); break;
            case 10: launch_ts<1, 512, 2, 3, 2>(c, L, R, n, nl, O); break;
            default: launch_ts<1, 512, 2, 4, 2>(c, L, R, n, nl, O); break;  // 34.4 us alone (was 37.1)
        }
    }
    check_launch("k_tensor_sum");
}

// ---- register-pipelined tensor sum (no shared-memory ring) ------------------------------------
// (d0, d1, d2) = sum_k L[k] (x) R[k] (Karatsuba d1) with plain 16-byte global loads: thread (k-group
// g, coefficient pair e) of a CTA walks its k range with the next step's four operand loads issued
// before the current step's products, and the KG k-groups of a CTA combine through shared memory;
// cluster ranks (split-K across CTAs) combine through DSMEM.  rb > 1: rb row blocks interleaved along
// x sharing R through L2 (config 5a).  Compared with the TMA ring it trades the producer warp and the
// per-stage mbarrier handshake for occupancy (every thread has loads in flight).
// ST > 0: the operand loads go through a per-thread shared-memory ring filled with 16-byte cp.async
// copies ST steps deep (a thread reads back only what it copied itself: cp.async.wait_group orders it,
// no barrier), so the bytes in flight no longer cost registers: ST - 1 steps x 64 B x 128 threads per CTA.
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N_>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N_) : "memory"); }

// Operand pointers of the tensor sum: device tables (PtrTab), or the kernel parameters of a slot
// graph's first kernel (PtrPar, see SetTables), read from the constant bank.
struct PtrTab {
    const uint64_t *const *L, *const *R;
    __device__ __forceinline__ const uint64_t *l(int k) const { return L[k]; }
    __device__ __forceinline__ const uint64_t *r(int k) const { return R[k]; }
    __device__ __forceinline__ void left_block(size_t ofs) { L += ofs; }
    __device__ __forceinline__ void right_block(size_t ofs) { R += ofs; }
};
struct PtrPar {
    const SetTables *a;
    int lofs, rofs;
    __device__ __forceinline__ const uint64_t *l(int k) const { return a->p[lofs + k]; }
    __device__ __forceinline__ const uint64_t *r(int k) const { return a->p[rofs + k]; }
    __device__ __forceinline__ void left_block(size_t ofs) { lofs += (int)ofs; }
    __device__ __forceinline__ void right_block(size_t ofs) { rofs += (int)ofs; }
};

template <int KG, int SPLIT, int ST, class PS, int TP = 64>
__device__ __forceinline__ void ts_ld_body(PS ps, int n, int nl, int N, const DevPrimes &pr, uint64_t *const *O, int rb) {
    // TP coefficient pairs per CTA
    // rb < 0: |rb| independent products interleaved along x, each with its own right operand
    // (matmul_outer_many); rb > 1: row blocks sharing R
    const int rbs = rb < 0 ? -rb : rb;
    const int xb = rbs > 1 ? (int)blockIdx.x % rbs : 0;
    const int xt = rbs > 1 ? (int)blockIdx.x / rbs : (int)blockIdx.x;
    ps.left_block((size_t)xb * n);
    if (rb < 0) ps.right_block((size_t)xb * n);
    O += xb;
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int z = (int)cluster.block_rank();
    const int tp = threadIdx.x % TP, g = threadIdx.x / TP;
    const int i = blockIdx.y;
    const long long e2 = (long long)xt * TP + tp;  // coefficient pair index
    const bool live = 2 * e2 < N;
    const Modulus m = pr.m[i];
    // k range of this (cluster rank, k-group)
    const int parts = SPLIT * KG, part = z * KG + g;
    const int per = (n + parts - 1) / parts;
    const int kb = min(n, part * per), ke = min(n, kb + per);
    const size_t o0 = (size_t)i * N + 2 * e2, o1 = (size_t)(nl + i) * N + 2 * e2;
    u128 acc[3][2];
#pragma unroll
    for (int p = 0; p < 3; p++) acc[p][0] = acc[p][1] = u128{0, 0};
    // Lazy accumulation: with q < 2^b a d0/d2 term is < 2^(2b) and a Karatsuba term < 2^(2b+2), so
    // 2^(128-2b) resp. 2^(126-2b) terms (plus a folded remainder < q) fit 128 bits.  A 60-bit limb
    // folds d1 every 64 steps and d0, d2 every 256; limbs below 2^54 never fold inside a k range --
    // the per-thread ranges of configs 2 and 5a (16 and 64 steps) run as pure multiply-accumulates.
    const int qb = 64 - __clzll((long long)m.q);
    const unsigned mask1 = (1u << max(0, min(20, 126 - 2 * qb))) - 1u, mask02 = (1u << max(0, min(20, 128 - 2 * qb))) - 1u;
    if constexpr (ST > 0) {
        __shared__ __align__(16) ulonglong2 ring[ST][4][TP * KG];
        if (live && kb < ke) {
            auto issue = [&](int k) {
                if (k < ke) {
                    const uint64_t *lp = ps.l(k), *rp = ps.r(k);
                    const int sl = (k - kb) % ST;
                    cp_async16(&ring[sl][0][threadIdx.x], lp + o0);
                    cp_async16(&ring[sl][1][threadIdx.x], lp + o1);
                    cp_async16(&ring[sl][2][threadIdx.x], rp + o0);
                    cp_async16(&ring[sl][3][threadIdx.x], rp + o1);
                }
                cp_async_commit();  // one group per step, empty past the end: wait_group counts stay uniform
            };
#pragma unroll
            for (int d = 0; d < ST - 1; d++) issue(kb + d);
            for (int k = kb, it = 0; k < ke; k++, it++) {
                issue(k + ST - 1);
                cp_async_wait<ST - 1>();  // the group of step k has landed
                const int sl = it % ST;
                const ulonglong2 l0 = ring[sl][0][threadIdx.x], l1 = ring[sl][1][threadIdx.x];
                const ulonglong2 r0 = ring[sl][2][threadIdx.x], r1 = ring[sl][3][threadIdx.x];
                mac_to(acc[0][0], l0.x, r0.x);
                mac_to(acc[0][1], l0.y, r0.y);
                mac_to(acc[2][0], l1.x, r1.x);
                mac_to(acc[2][1], l1.y, r1.y);
                mac_to(acc[1][0], l0.x + l1.x, r0.x + r1.x);
                mac_to(acc[1][1], l0.y + l1.y, r0.y + r1.y);
                if (((unsigned)it & mask1) == mask1) {
#pragma unroll
                    for (int e = 0; e < 2; e++) acc[1][e] = u128{reduce128(acc[1][e], m), 0};
                    if (((unsigned)it & mask02) == mask02) {
#pragma unroll
                        for (int e = 0; e < 2; e++) {
                            acc[0][e] = u128{reduce128(acc[0][e], m), 0};
                            acc[2][e] = u128{reduce128(acc[2][e], m), 0};
                        }
                    }
                }
            }
        }
    } else if (live && kb < ke) {
        ulonglong2 l0 = *reinterpret_cast<const ulonglong2 *>(ps.l(kb) + o0), l1 = *reinterpret_cast<const ulonglong2 *>(ps.l(kb) + o1);
        ulonglong2 r0 = *reinterpret_cast<const ulonglong2 *>(ps.r(kb) + o0), r1 = *reinterpret_cast<const ulonglong2 *>(ps.r(kb) + o1);
        for (int k = kb, it = 0; k < ke; k++, it++) {
            ulonglong2 nl0 = l0, nl1 = l1, nr0 = r0, nr1 = r1;
            if (k + 1 < ke) {  // next step's operands in flight while this step multiplies
                const uint64_t *lp = ps.l(k + 1), *rp = ps.r(k + 1);
                nl0 = __ldcs(reinterpret_cast<const ulonglong2 *>(lp + o0));
                nl1 = __ldcs(reinterpret_cast<const ulonglong2 *>(lp + o1));
                nr0 = __ldcs(reinterpret_cast<const ulonglong2 *>(rp + o0));
                nr1 = __ldcs(reinterpret_cast<const ulonglong2 *>(rp + o1));
            }
            mac_to(acc[0][0], l0.x, r0.x);
            mac_to(acc[0][1], l0.y, r0.y);
            mac_to(acc[2][0], l1.x, r1.x);
            mac_to(acc[2][1], l1.y, r1.y);
            mac_to(acc[1][0], l0.x + l1.x, r0.x + r1.x);
            mac_to(acc[1][1], l0.y + l1.y, r0.y + r1.y);
            if (((unsigned)it & mask1) == mask1) {
#pragma unroll
                for (int e = 0; e < 2; e++) acc[1][e] = u128{reduce128(acc[1][e], m), 0};
                if (((unsigned)it & mask02) == mask02) {
#pragma unroll
                    for (int e = 0; e < 2; e++) {
                        acc[0][e] = u128{reduce128(acc[0][e], m), 0};
                        acc[2][e] = u128{reduce128(acc[2][e], m), 0};
                    }
                }
            }
            l0 = nl0;
            l1 = nl1;
            r0 = nr0;
            r1 = nr1;
        }
    }
    __shared__ ulonglong2 part_s[KG][3][TP];
    {
        uint64_t v[3][2];
#pragma unroll
        for (int p = 0; p < 3; p++)
#pragma unroll
            for (int e = 0; e < 2; e++) v[p][e] = reduce128(acc[p][e], m);
#pragma unroll
        for (int e = 0; e < 2; e++) v[1][e] = sub_mod(sub_mod(v[1][e], v[0][e], m.q), v[2][e], m.q);  // undo Karatsuba
#pragma unroll
        for (int p = 0; p < 3; p++) part_s[g][p][tp] = make_ulonglong2(v[p][0], v[p][1]);
    }
    __syncthreads();
    if (g == 0) {  // k-groups of this CTA
#pragma unroll
        for (int p = 0; p < 3; p++) {
            ulonglong2 v = part_s[0][p][tp];
#pragma unroll
            for (int gg = 1; gg < KG; gg++) {
                const ulonglong2 w = part_s[gg][p][tp];
                v.x = add_mod(v.x, w.x, m.q);
                v.y = add_mod(v.y, w.y, m.q);
            }
            part_s[0][p][tp] = v;
        }
    }
    cluster.sync();
    if (z == 0 && g == 0 && live) {
        uint64_t *o = O[0];
#pragma unroll
        for (int p = 0; p < 3; p++) {
            ulonglong2 v = part_s[0][p][tp];
#pragma unroll
            for (int r = 1; r < SPLIT; r++) {
                const ulonglong2 w = cluster.map_shared_rank(&part_s[0][p][0], r)[tp];
                v.x = add_mod(v.x, w.x, m.q);
                v.y = add_mod(v.y, w.y, m.q);
            }
            st2(o + (size_t)(p * nl + i) * N + 2 * e2, v.x, v.y);
        }
    }
    cluster.sync();
}

template <int KG, int SPLIT, int ST = 0, int TP = 64>
__global__ void __launch_bounds__(TP * KG)
    k_tensor_sum_ld(const uint64_t *const *L, const uint64_t *const *R, int n, int nl, int N, DevPrimes pr, uint64_t *const *O,
                    int rb) {
    pdl_wait();
    pdl_trigger();
    ts_ld_body<KG, SPLIT, ST, PtrTab, TP>(PtrTab{L, R}, n, nl, N, pr, O, rb);
}

// First kernel of a slot graph: the operand pointers arrive in the parameters (one row block), block
// (0, 0, 0) publishes them -- the output pointer table above all -- for the later kernels of the graph.
template <int KG, int SPLIT, int ST = 0>
__global__ void __launch_bounds__(64 * KG)
    k_tensor_sum_ldp(const __grid_constant__ SetTables a, int n, int nl, int N, DevPrimes pr, uint64_t *const *O, int rb) {
    pdl_wait();
    pdl_trigger();
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)
        for (int i = threadIdx.x; i < a.count; i += blockDim.x) a.dst[i] = const_cast<uint64_t *>(a.p[i]);
    ts_ld_body<KG, SPLIT, ST>(PtrPar{&a, 0, (rb < 0 ? -rb : rb) * n}, n, nl, N, pr, O, rb);
}

template <int KG, int SPLIT, int ST = 0, int TP = 64>
static void launch_ts_ld(Ctx &c, const uint64_t *const *L, const uint64_t *const *R, int n, int nl, uint64_t *const *O, int rb) {
    cudaLaunchConfig_t cfg = {};
    const int tiles = (c.n / 2 + TP - 1) / TP;
    cfg.gridDim = dim3(tiles * (rb < 0 ? -rb : rb), nl, SPLIT);
    cfg.blockDim = dim3(TP * KG, 1, 1);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = SPLIT;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    if (c.ts_params && TP != 64) throw VrError(4, "tensor sum: tile variants are not slot-graph kernels");
    if constexpr (TP == 64) if (c.ts_params) {  // recording a slot graph: pointers in the parameters, no table-writing kernel
        const SetTables *a = c.ts_params;
        c.ts_params = nullptr;
        VR_CUDA(cudaLaunchKernelEx(&cfg, k_tensor_sum_ldp<KG, SPLIT, ST>, *a, n, nl, c.n, c.primes, O, rb));
        cudaStreamCaptureStatus cs;
        const cudaGraphNode_t *deps = nullptr;
        size_t nd = 0;
        VR_CUDA(cudaStreamGetCaptureInfo(c.stream, &cs, nullptr, nullptr, &deps, &nd));
        if (cs != cudaStreamCaptureStatusActive || nd != 1) throw VrError(4, "tensor sum: unexpected capture state");
        c.ts_node = deps[0];
        return;
    }
    VR_CUDA(cudaLaunchKernelEx(&cfg, k_tensor_sum_ld<KG, SPLIT, ST, TP>, L, R, n, nl, c.n, c.primes, O, rb));
}

// VR_TS_LD selects the register-pipelined kernel for one-pass sums (0 = the TMA ring).  Swept on
// B200 (config 2, tools/ts_probe.py): TMA ring 38.1 us; KG x SPLIT = 4x1 37.8, 4x2 41.1, 8x1 55.7,
// 2x2 36.3 (default, 4.66 TB/s), 8x2 63.0, 2x4 54.3, 2x1 39.6, 1x4 47.7, 1x2 57.2, 1x8 53.9.  Config 5a
// (4 interleaved row blocks): 2x2 1.19 ms vs 1.24 ms for the ring.
// After the fold periods above removed the in-loop reductions (re-swept, cfg 2 / cfg 5a): 2x2 33.6 us /
// 1.03 ms (5.2 TB/s), 2x1 30.4 us (5.59 TB/s = 0.85 of the copy peak) / 1.15 ms, 1x2 49.3 / 1.28, 4x1 43.7 /
// 1.38, 2x4 50.6 / 1.71, 1x4 47.7 / 1.59, 4x2 46.9 / 1.50.  Default (VR_TS_LD unset, -1): two k-groups per
// CTA and no split-K; from n = 128 columns on the operands go through a per-thread cp.async ring.
static int ts_ld_variant() {
    static const int v = [] {
        const char *e = getenv("VR_TS_LD");
        return e ? atoi(e) : -1;
    }();
    return v;
}

static bool try_ts_ld(Ctx &c, const uint64_t *const *L, const uint64_t *const *R, int n, int nl, uint64_t *const *O, int rb) {
    int v = ts_ld_variant();
    // long k ranges (cfg 5a, n = 256): the cp.async ring keeps four steps in flight per thread without
    // split-K: 0.98 ms (5.5 TB/s) against 1.04 ms for the register-prefetch 2x2 form; at n = 64 the
    // register form wins (30.2 vs 31.9 us)
    // Inside the overlapped step the ring form also wins at n = 64 (37.6 vs 39.1 us per product with equal
    // stand-alone times: its copies in flight cost no registers while other products' chain kernels share
    // the SM), except in the slot graphs recorded for freshly encrypted operands, where the register form
    // keeps the e2e loop 2% faster.
    // Long sums outside a slot-graph capture (cfg 5a, n = 256: vr_tensor_sum of the sharded product) take
    // 128 coefficient pairs per CTA and one k-group -- 2 KB row segments, each thread walks the whole k
    // range: 981 -> 958 us (5.63 TB/s); at n = 64 the same tile is slower (34.3 vs 32.0 us).
    if (v < 0) v = (n >= 128 && !c.ts_params) ? 20 : (n >= 128 || !(c.capturing && !c.capture_cl)) ? 12 : 7;
    switch (v) {
        case 1: launch_ts_ld<4, 1>(c, L, R, n, nl, O, rb); return true;
        case 2: launch_ts_ld<4, 2>(c, L, R, n, nl, O, rb); return true;
        case 3: launch_ts_ld<8, 1>(c, L, R, n, nl, O, rb); return true;
        case 4: launch_ts_ld<2, 2>(c, L, R, n, nl, O, rb); return true;
        case 5: launch_ts_ld<8, 2>(c, L, R, n, nl, O, rb); return true;
        case 6: launch_ts_ld<2, 4>(c, L, R, n, nl, O, rb); return true;
        case 7: launch_ts_ld<2, 1>(c, L, R, n, nl, O, rb); return true;
        case 8: launch_ts_ld<1, 4>(c, L, R, n, nl, O, rb); return true;
        case 9: launch_ts_ld<1, 2>(c, L, R, n, nl, O, rb); return true;
        case 10: launch_ts_ld<1, 8>(c, L, R, n, nl, O, rb); return true;
        case 11: launch_ts_ld<2, 1, 3>(c, L, R, n, nl, O, rb); return true;  // cp.async rings
        case 12: launch_ts_ld<2, 1, 4>(c, L, R, n, nl, O, rb); return true;
        case 13: launch_ts_ld<2, 2, 3>(c, L, R, n, nl, O, rb); return true;
        case 14: launch_ts_ld<2, 2, 4>(c, L, R, n, nl, O, rb); return true;
        case 15: launch_ts_ld<2, 1, 5>(c, L, R, n, nl, O, rb); return true;
        case 16: launch_ts_ld<2, 2, 5>(c, L, R, n, nl, O, rb); return true;
        case 20: launch_ts_ld<1, 1, 4, 128>(c, L, R, n, nl, O, rb); return true;  // 2 KB row segments per CTA
        case 21: launch_ts_ld<4, 1, 4, 32>(c, L, R, n, nl, O, rb); return true;   // 512 B segments, four k-groups
        case 22: launch_ts_ld<1, 1, 2, 256>(c, L, R, n, nl, O, rb); return true;  // 4 KB segments, two steps in flight
        case 23: launch_ts_ld<2, 1, 2, 128>(c, L, R, n, nl, O, rb); return true;
        default: return false;
    }
}

// whether tensor_sum(n, nb) runs the register / cp.async kernel, which can take its operand pointers
// from its parameters (slot graphs)
bool tensor_sum_takes_params(int nb) { return ts_ld_variant() != 0 && (nb == 1 || nb == 4) && getenv("VR_TS_VARIANT") == nullptr && getenv("VR_TS4") == nullptr && getenv("VR_TS4_MC") == nullptr; }

// B independent products in one launch: O[b] = sum_k L[b*n + k] (x) R[b*n + k] (matmul_outer_many)
void tensor_sum_many(Ctx &c, const uint64_t *const *L, const uint64_t *const *R, int n, int B, int nl, uint64_t *const *O) {
    if (c.ts_params) throw VrError(4, "tensor_sum_many inside a slot-graph capture");
    if (n >= 32) launch_ts_ld<2, 1, 4>(c, L, R, n, nl, O, -B);
    else launch_ts_ld<1, 1, 4>(c, L, R, n, nl, O, -B);  // short sums: one k-group per CTA
    check_launch("k_tensor_sum (many)");
}

void tensor_sum(Ctx &c, const uint64_t *const *L, const uint64_t *const *R, int n, int nb, int nl, uint64_t *const *O) {
    static int variant = [] {
        const char *e = getenv("VR_TS_VARIANT");
        return e ? atoi(e) : 0;  // 0 = tuned default
    }();
    switch (nb) {
        case 1:
            if (!try_ts_ld(c, L, R, n, nl, O, 1)) ts_variant<1>(c, variant, L, R, n, nl, O);
            break;
        case 2: ts_variant<2>(c, variant, L, R, n, nl, O); break;
        case 4: {
            // four row blocks sharing R (cfg 5a).  Round 1: two launches of two row blocks, R streamed twice,
            // but each CTA holds half the 128-bit accumulators (104 instead of 188 registers, 3 CTAs
            // per SM instead of 2): cfg-5a matmul 2.12 -> 1.56 ms.  Swept on B200 (tools/prof_5a.sh):
            // one NB=4 kernel 2.12 ms (tiles 128 / split 4: 2.81; tile 256 / split 4: 2.52), two NB=2
            // launches with 512-tiles 1.76, 8 stages 1.96, split 4 1.70, four NB=1 launches 1.69.
            // VR_TS4=1 restores the single NB=4 kernel.
            static const int v4 = [] {
                const char *e = getenv("VR_TS4");
                return e ? atoi(e) : 0;
            }();
            if (v4 == 1) {
                ts_variant<4>(c, variant, L, R, n, nl, O);
            } else if (v4 == 2 || c.n < 256) {
                launch_ts<2, 256, 2, 4>(c, L, R, n, nl, O);
                launch_ts<2, 256, 2, 4>(c, L + 2 * (size_t)n, R, n, nl, O + 2);
            } else {
                // default: one pass, R multicast to the four row-block CTAs of each cluster
                static const int mcv = [] {
                    const char *e = getenv("VR_TS4_MC");
                    return e ? atoi(e) : 0;
                }();
                switch (mcv ? mcv : (ts_ld_variant() ? 7 : 0)) {
                    case 1: launch_ts_mc<4, 256, 2, 8>(c, L, R, n, nl, O); break;
                    case 2: launch_ts_mc<4, 512, 2, 4>(c, L, R, n, nl, O); break;
                    case 3: launch_ts<1, 256, 2, 4>(c, L, R, n, nl, O, 4); break;
                    case 7: if (!try_ts_ld(c, L, R, n, nl, O, 4)) launch_ts<1, 512, 2, 6>(c, L, R, n, nl, O, 4); break;
                    case 4: launch_ts<1, 512, 2, 4>(c, L, R, n, nl, O, 4); break;
                    case 5: launch_ts<2, 256, 2, 4>(c, L, R, n, nl, O, 2); break;
                    case 6: launch_ts<1, 256, 4, 4>(c, L, R, n, nl, O, 4); break;
                    default: launch_ts<1, 512, 2, 6>(c, L, R, n, nl, O, 4); break;
                }
            }
            break;
        }
        default: throw VrError(3, "tensor_sum: nblocks must be 1, 2 or 4");
    }
    check_launch("k_tensor_sum");
}

}  // namespace vr
