// ring.cu -- RNS elementwise kernels (add/sub/tensor/plain & scalar products,
// Galois permutation, level drop) and the fused column-ciphertext tensor-sum
// that realises matmul_outer's hot loop (multicipher.py:100-102).
//
// All kernels are HBM-bound streaming passes over [poly][limb][N] uint64
// arrays; each thread handles two adjacent coefficients with 128-bit loads so
// a warp moves 512 contiguous bytes per access.
#include <cooperative_groups.h>

#include "ring.cuh"

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

__global__ void k_add_const(uint64_t *const *C, int count, int nl, int N, LimbScalars s, DevPrimes pr) {
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
    const long long pair = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (pair >= (long long)count * polys * nl_out * (N / 2)) return;
    Idx x;
    decompose(pair, polys, nl_out, N, x);
    ulonglong2 a = ld2(C[x.ct] + ((size_t)x.poly * nl_in + x.limb + limb0) * N + x.k);
    st2(O[x.ct] + ((size_t)x.poly * nl_out + x.limb) * N + x.k, a.x, a.y);
}

__global__ void k_mod_fixup(uint64_t *data, long long count_polys, int nl, int N, DevPrimes pr) {
    const long long pair = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (pair >= count_polys * nl * (N / 2)) return;
    Idx x;
    decompose(pair, 1, nl, N, x);
    const Modulus m = pr.m[x.limb];
    uint64_t *p = data + ((size_t)x.ct * nl + x.limb) * N + x.k;
    ulonglong2 a = ld2(p);
    st2(p, reduce64(a.x, m), reduce64(a.y, m));
}

// Fused sum_k tensor(L[b][k], R[k]) for NB row blocks sharing the right operand.
// Grid (coefficient tiles, limbs, SPLIT): the SPLIT CTAs of a thread-block
// cluster walk disjoint quarters of the k range for the same 256 coefficients,
// accumulate 64x64->128-bit products (folded mod q every 8 terms), reduce
// their partials mod q and combine them through distributed shared memory;
// cluster rank 0 writes the degree-2 result.  R is read once per block group.
constexpr int TS_THREADS = 128, TS_SPLIT = 4;

template <int NB>
__global__ void __cluster_dims__(1, 1, TS_SPLIT) __launch_bounds__(TS_THREADS)
    k_tensor_sum(const uint64_t *const *L, const uint64_t *const *R, int n, int nl, int N, DevPrimes pr, uint64_t *const *O) {
    __shared__ ulonglong2 part[NB * 3][TS_THREADS];
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int k = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
    const int i = blockIdx.y;
    const int z = (int)cluster.block_rank();
    const bool live = k < N;
    const Modulus m = pr.m[i];
    const size_t o0 = (size_t)i * N + k, o1 = (size_t)(nl + i) * N + k;
    const int per = (n + TS_SPLIT - 1) / TS_SPLIT;
    const int tb = z * per, te = min(n, tb + per);
    u128 acc[NB][3][2];
#pragma unroll
    for (int b = 0; b < NB; b++)
#pragma unroll
        for (int p = 0; p < 3; p++)
#pragma unroll
            for (int e = 0; e < 2; e++) acc[b][p][e] = u128{0, 0};
    if (live) {
        for (int t0 = tb; t0 < te; t0 += 8) {
            const int tend = min(te, t0 + 8);
#pragma unroll 4
            for (int t = t0; t < tend; t++) {
                const uint64_t *r = R[t];
                const ulonglong2 r0 = ld2(r + o0), r1 = ld2(r + o1);
#pragma unroll
                for (int b = 0; b < NB; b++) {
                    const uint64_t *l = L[b * n + t];
                    const ulonglong2 l0 = ld2(l + o0), l1 = ld2(l + o1);
                    mac_to(acc[b][0][0], l0.x, r0.x);
                    mac_to(acc[b][0][1], l0.y, r0.y);
                    mac_to(acc[b][1][0], l0.x, r1.x);
                    mac_to(acc[b][1][1], l0.y, r1.y);
                    mac_to(acc[b][1][0], l1.x, r0.x);
                    mac_to(acc[b][1][1], l1.y, r0.y);
                    mac_to(acc[b][2][0], l1.x, r1.x);
                    mac_to(acc[b][2][1], l1.y, r1.y);
                }
            }
            if (tend < te) {
#pragma unroll
                for (int b = 0; b < NB; b++)
#pragma unroll
                    for (int p = 0; p < 3; p++)
#pragma unroll
                        for (int e = 0; e < 2; e++) acc[b][p][e] = u128{reduce128(acc[b][p][e], m), 0};
            }
        }
    }
#pragma unroll
    for (int b = 0; b < NB; b++)
#pragma unroll
        for (int p = 0; p < 3; p++)
            part[b * 3 + p][threadIdx.x] = make_ulonglong2(reduce128(acc[b][p][0], m), reduce128(acc[b][p][1], m));
    cluster.sync();
    if (z == 0 && live) {
#pragma unroll
        for (int b = 0; b < NB; b++) {
            uint64_t *o = O[b];
#pragma unroll
            for (int p = 0; p < 3; p++) {
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

constexpr int TB = 256;

}  // namespace

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
    k_binop<<<nblocks(pairs, TB), TB, 0, c.stream>>>(A, B, O, count, polys, nl, c.n, op, c.primes);
    check_launch("k_binop");
}

void tensor(Ctx &c, const uint64_t *const *A, const uint64_t *const *B, uint64_t *const *O, int count, int nl) {
    const long long pairs = (long long)count * nl * (c.n / 2);
    k_tensor<<<nblocks(pairs, TB), TB, 0, c.stream>>>(A, B, O, count, nl, c.n, c.primes);
    check_launch("k_tensor");
}

void mul_plain(Ctx &c, const uint64_t *const *C, const uint64_t *const *P, uint64_t *const *O, int count, int polys, int nl,
               int shared_pt) {
    const long long pairs = (long long)count * polys * nl * (c.n / 2);
    k_mul_plain<<<nblocks(pairs, TB), TB, 0, c.stream>>>(C, P, O, count, polys, nl, c.n, shared_pt, c.primes);
    check_launch("k_mul_plain");
}

void mul_scalar(Ctx &c, const uint64_t *const *C, uint64_t *const *O, int count, int polys, int nl, const LimbScalars &s) {
    const long long pairs = (long long)count * polys * nl * (c.n / 2);
    k_mul_scalar<<<nblocks(pairs, TB), TB, 0, c.stream>>>(C, O, count, polys, nl, c.n, s, c.primes);
    check_launch("k_mul_scalar");
}

void axpy(Ctx &c, uint64_t *const *O, const uint64_t *const *B, int count, int polys, int nl, int nlb, const LimbScalars &s) {
    const long long pairs = (long long)count * polys * nl * (c.n / 2);
    k_axpy<<<nblocks(pairs, TB), TB, 0, c.stream>>>(O, B, count, polys, nl, nlb, c.n, s, c.primes);
    check_launch("k_axpy");
}

void add_const(Ctx &c, uint64_t *const *C, int count, int nl, const LimbScalars &s) {
    const long long pairs = (long long)count * nl * (c.n / 2);
    k_add_const<<<nblocks(pairs, TB), TB, 0, c.stream>>>(C, count, nl, c.n, s, c.primes);
    check_launch("k_add_const");
}

void permute(Ctx &c, const uint64_t *const *C, uint64_t *const *O, int count, int polys, int nl, uint32_t g) {
    const long long el = (long long)count * polys * nl * c.n;
    k_permute<<<nblocks(el, TB), TB, 0, c.stream>>>(C, O, count, polys, nl, c.log_n, g);
    check_launch("k_permute");
}

void copy_limbs(Ctx &c, const uint64_t *const *C, uint64_t *const *O, int count, int polys, int nl_in, int nl_out, int limb0) {
    const long long pairs = (long long)count * polys * nl_out * (c.n / 2);
    if (!pairs) return;
    k_copy_limbs<<<nblocks(pairs, TB), TB, 0, c.stream>>>(C, O, count, polys, nl_in, nl_out, limb0, c.n);
    check_launch("k_copy_limbs");
}

void mod_fixup(Ctx &c, uint64_t *data, long long count_polys, int nl) {
    const long long pairs = count_polys * nl * (c.n / 2);
    k_mod_fixup<<<nblocks(pairs, TB), TB, 0, c.stream>>>(data, count_polys, nl, c.n, c.primes);
    check_launch("k_mod_fixup");
}

void tensor_sum(Ctx &c, const uint64_t *const *L, const uint64_t *const *R, int n, int nb, int nl, uint64_t *const *O) {
    dim3 grid(nblocks(c.n / 2, TS_THREADS), nl, TS_SPLIT);
    switch (nb) {
        case 1: k_tensor_sum<1><<<grid, TS_THREADS, 0, c.stream>>>(L, R, n, nl, c.n, c.primes, O); break;
        case 2: k_tensor_sum<2><<<grid, TS_THREADS, 0, c.stream>>>(L, R, n, nl, c.n, c.primes, O); break;
        case 4: k_tensor_sum<4><<<grid, TS_THREADS, 0, c.stream>>>(L, R, n, nl, c.n, c.primes, O); break;
        default: throw VrError(3, "tensor_sum: nblocks must be 1, 2 or 4");
    }
    check_launch("k_tensor_sum");
}

}  // namespace vr
