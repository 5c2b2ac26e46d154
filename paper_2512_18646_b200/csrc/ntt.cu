// ntt.cu -- batched negacyclic NTT / INTT over RNS limbs for sm_100a.
//
// Transform definition (identical to oracle/ckks_oracle.c orc_ntt/orc_intt):
//   forward  = Cooley-Tukey, natural in -> bit-reversed out, stage g (m = 2^g)
//              pairs elements at distance N >> (g+1) with twiddle
//              psi_br[2^g + (E >> (logN - g))]  (E = index of the upper element);
//   inverse  = Gentleman-Sande with psi^-1 in the same indexing, times N^-1.
//
// Kernel structure.  N = N1 * N2.  Pass 1 runs stages g < log N1: every
// "column" {c + r*N2} is an independent N1-point sub-transform, a CTA stages
// 16 adjacent columns (128-byte rows, coalesced) in shared memory.  Pass 2
// runs the remaining stages inside contiguous N2-element rows.  Inside a pass
// each thread owns 8 elements and performs up to three stages in registers
// (radix-8) between shared-memory exchanges.  Butterflies are Harvey-lazy
// (values in [0,4q) forward / [0,2q) inverse, Shoup twiddle products); the
// last pass writes fully reduced values.  The inverse folds N^-1 into its
// final stage.  Small N (< 2048) runs as a single pass, N <= 32 by a scalar
// per-thread kernel (test-only sizes).
#include "vrhe_internal.cuh"

namespace vr {

namespace {

__device__ __forceinline__ bool locate(const NttBatch &b, int t, int N, uint64_t *&ptr, int &pidx) {
    int g = t / b.group, r = t - g * b.group;
    if (b.skip_diag > 0 && r == g % b.skip_diag) return false;
    ptr = b.data + (long long)g * b.gstride + (long long)r * N;
    pidx = r < b.nq ? b.poff + r : b.pspecial;
    return true;
}

template <bool COLS>
__device__ __forceinline__ int sidx(int j, int L, int T, int TPC) {
    if (COLS) return L * TPC + j;
    return j * T + (L ^ ((L >> 4) & 15));
}

__device__ __forceinline__ void bf_fwd(uint64_t &X, uint64_t &Y, uint64_t w, uint64_t wsh, uint64_t q, uint64_t q2) {
    uint64_t x = X >= q2 ? X - q2 : X;
    uint64_t t = mul_shoup_lazy(Y, w, wsh, q);
    X = x + t;
    Y = x - t + q2;
}

__device__ __forceinline__ void bf_inv(uint64_t &X, uint64_t &Y, uint64_t w, uint64_t wsh, uint64_t q, uint64_t q2) {
    uint64_t t = X + Y;
    t = t >= q2 ? t - q2 : t;
    uint64_t u = X - Y + q2;
    Y = mul_shoup_lazy(u, w, wsh, q);
    X = t;
}

struct PassArgs {
    int logN, s0, s1, TPC;
    int first, last;  // first pass reads raw input, last pass writes reduced output
};

template <bool COLS, int R>
__device__ __forceinline__ void group_fwd(uint64_t *sm, int j, int sub, int s, int logT, int T, int TPC, int s0, int hi,
                                          uint64_t q, const uint64_t *__restrict__ W, const uint64_t *__restrict__ Wsh) {
    constexpr int E2 = 1 << R, U = 8 >> R;
    const int logd = logT - s - R, d = 1 << logd;
    const uint64_t q2 = 2 * q;
#pragma unroll
    for (int v = 0; v < U; v++) {
        const int uid = sub * U + v;
        const int base = ((uid >> logd) << (logd + R)) | (uid & (d - 1));
        uint64_t x[E2];
#pragma unroll
        for (int w = 0; w < E2; w++) x[w] = sm[sidx<COLS>(j, base + w * d, T, TPC)];
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int g = s0 + s + r, half = E2 >> (r + 1), shift = logT - (s + r);
#pragma unroll
            for (int w = 0; w < E2; w++) {
                if (w & half) continue;
                const int idx = (1 << g) + (hi << (g - s0)) + ((base + w * d) >> shift);
                bf_fwd(x[w], x[w + half], __ldg(W + idx), __ldg(Wsh + idx), q, q2);
            }
        }
#pragma unroll
        for (int w = 0; w < E2; w++) sm[sidx<COLS>(j, base + w * d, T, TPC)] = x[w];
    }
}

template <bool COLS, int R>
__device__ __forceinline__ void group_inv(uint64_t *sm, int j, int sub, int s, int logT, int T, int TPC, int s0, int hi,
                                          uint64_t q, const uint64_t *__restrict__ W, const uint64_t *__restrict__ Wsh,
                                          const NttConst &nc) {
    constexpr int E2 = 1 << R, U = 8 >> R;
    const int logd = logT - s - R, d = 1 << logd;
    const uint64_t q2 = 2 * q;
#pragma unroll
    for (int v = 0; v < U; v++) {
        const int uid = sub * U + v;
        const int base = ((uid >> logd) << (logd + R)) | (uid & (d - 1));
        uint64_t x[E2];
#pragma unroll
        for (int w = 0; w < E2; w++) x[w] = sm[sidx<COLS>(j, base + w * d, T, TPC)];
#pragma unroll
        for (int r = R - 1; r >= 0; r--) {
            const int g = s0 + s + r, half = E2 >> (r + 1), shift = logT - (s + r);
#pragma unroll
            for (int w = 0; w < E2; w++) {
                if (w & half) continue;
                if (g == 0) {
                    // final GS stage with N^-1 folded in
                    uint64_t X = x[w], Y = x[w + half];
                    x[w] = mul_shoup_lazy(X + Y, nc.ninv, nc.ninv_sh, q);
                    x[w + half] = mul_shoup_lazy(X - Y + q2, nc.w0n, nc.w0n_sh, q);
                } else {
                    const int idx = (1 << g) + (hi << (g - s0)) + ((base + w * d) >> shift);
                    bf_inv(x[w], x[w + half], __ldg(W + idx), __ldg(Wsh + idx), q, q2);
                }
            }
        }
#pragma unroll
        for (int w = 0; w < E2; w++) sm[sidx<COLS>(j, base + w * d, T, TPC)] = x[w];
    }
}

template <bool INV, bool COLS>
__global__ void __launch_bounds__(512) ntt_pass_kernel(NttBatch b, PassArgs a, DevPrimes pr, const uint64_t *__restrict__ tw,
                                                       const uint64_t *__restrict__ twsh, const NttConst *__restrict__ ncs) {
    extern __shared__ uint64_t sm[];
    const int logN = a.logN, N = 1 << logN, s0 = a.s0, logT = a.s1 - a.s0, T = 1 << logT;
    const int lo_bits = logN - a.s1, TPC = a.TPC;
    const int chunks = (N >> logT) / TPC;
    const int t = blockIdx.x / chunks, chunk = blockIdx.x - t * chunks;
    uint64_t *ptr;
    int pidx;
    if (!locate(b, t, N, ptr, pidx)) return;
    const uint64_t q = pr.m[pidx].q;
    const uint64_t *W = tw + (size_t)pidx * N, *Wsh = twsh + (size_t)pidx * N;
    const int tile0 = chunk * TPC, lomask = (1 << lo_bits) - 1;

    for (int idx = threadIdx.x; idx < TPC * T; idx += blockDim.x) {
        int j, mid;
        if (COLS) { mid = idx / TPC; j = idx - mid * TPC; }
        else { j = idx >> logT; mid = idx & (T - 1); }
        const int tile = tile0 + j, hi = tile >> lo_bits, lo = tile & lomask;
        const long long E = ((long long)hi << (logN - s0)) | ((long long)mid << lo_bits) | lo;
        sm[sidx<COLS>(j, mid, T, TPC)] = ptr[E];
    }
    __syncthreads();

    const int tpt = T >> 3;
    int j, sub;
    if (COLS) { j = threadIdx.x % TPC; sub = threadIdx.x / TPC; }
    else { j = threadIdx.x / tpt; sub = threadIdx.x - j * tpt; }
    const int hi = (tile0 + j) >> lo_bits;
    if (!INV) {
        for (int s = 0; s < logT;) {
            const int R = min(3, logT - s);
            if (R == 3) group_fwd<COLS, 3>(sm, j, sub, s, logT, T, TPC, s0, hi, q, W, Wsh);
            else if (R == 2) group_fwd<COLS, 2>(sm, j, sub, s, logT, T, TPC, s0, hi, q, W, Wsh);
            else group_fwd<COLS, 1>(sm, j, sub, s, logT, T, TPC, s0, hi, q, W, Wsh);
            s += R;
            __syncthreads();
        }
    } else {
        const NttConst nc = ncs[pidx];
        // same grouping as forward, traversed backwards
        int starts[8], rs[8], ng = 0;
        for (int s = 0; s < logT;) { const int R = min(3, logT - s); starts[ng] = s; rs[ng] = R; ng++; s += R; }
        for (int gi = ng - 1; gi >= 0; gi--) {
            const int s = starts[gi], R = rs[gi];
            if (R == 3) group_inv<COLS, 3>(sm, j, sub, s, logT, T, TPC, s0, hi, q, W, Wsh, nc);
            else if (R == 2) group_inv<COLS, 2>(sm, j, sub, s, logT, T, TPC, s0, hi, q, W, Wsh, nc);
            else group_inv<COLS, 1>(sm, j, sub, s, logT, T, TPC, s0, hi, q, W, Wsh, nc);
            __syncthreads();
        }
    }

    const uint64_t q2 = 2 * q;
    for (int idx = threadIdx.x; idx < TPC * T; idx += blockDim.x) {
        int jj, mid;
        if (COLS) { mid = idx / TPC; jj = idx - mid * TPC; }
        else { jj = idx >> logT; mid = idx & (T - 1); }
        const int tile = tile0 + jj, h = tile >> lo_bits, lo = tile & lomask;
        const long long E = ((long long)h << (logN - s0)) | ((long long)mid << lo_bits) | lo;
        uint64_t v = sm[sidx<COLS>(jj, mid, T, TPC)];
        if (a.last) {
            if (!INV) v = v >= q2 ? v - q2 : v;
            v = v >= q ? v - q : v;
        }
        ptr[E] = v;
    }
}

// scalar fallback for N <= 32 (test-only parameter sets)
__global__ void ntt_tiny_kernel(NttBatch b, int logN, int inv, DevPrimes pr, const uint64_t *__restrict__ tw,
                                const uint64_t *__restrict__ twsh, const NttConst *__restrict__ ncs) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= b.count) return;
    const int N = 1 << logN;
    uint64_t *a;
    int pidx;
    if (!locate(b, t, N, a, pidx)) return;
    const uint64_t q = pr.m[pidx].q;
    const uint64_t *w = tw + (size_t)pidx * N, *wsh = twsh + (size_t)pidx * N;
    if (!inv) {
        int tt = N;
        for (int m = 1; m < N; m <<= 1) {
            tt >>= 1;
            for (int i = 0; i < m; i++)
                for (int j = 2 * i * tt; j < 2 * i * tt + tt; j++) {
                    uint64_t u = a[j], v = mul_shoup(a[j + tt], w[m + i], wsh[m + i], q);
                    a[j] = add_mod(u, v, q);
                    a[j + tt] = sub_mod(u, v, q);
                }
        }
    } else {
        int tt = 1;
        for (int m = N; m > 1; m >>= 1) {
            int h = m >> 1, j1 = 0;
            for (int i = 0; i < h; i++) {
                for (int j = j1; j < j1 + tt; j++) {
                    uint64_t u = a[j], v = a[j + tt];
                    a[j] = add_mod(u, v, q);
                    a[j + tt] = mul_shoup(sub_mod(u, v, q), w[h + i], wsh[h + i], q);
                }
                j1 += 2 * tt;
            }
            tt <<= 1;
        }
        const NttConst nc = ncs[pidx];
        for (int j = 0; j < N; j++) a[j] = mul_shoup(a[j], nc.ninv, nc.ninv_sh, q);
    }
}

template <bool INV, bool COLS>
void launch_pass(Ctx &c, const NttBatch &b, const PassArgs &a) {
    const int T = 1 << (a.s1 - a.s0);
    const int chunks = (c.n >> (a.s1 - a.s0)) / a.TPC;
    const int threads = a.TPC * (T >> 3);
    const size_t smem = (size_t)a.TPC * T * sizeof(uint64_t);
    const unsigned blocks = (unsigned)b.count * chunks;
    ntt_pass_kernel<INV, COLS><<<blocks, threads, smem, c.stream>>>(b, a, c.primes, INV ? c.itw : c.tw,
                                                                    INV ? c.itw_sh : c.tw_sh, c.ntt_const);
    check_launch("ntt_pass_kernel");
}

void run(Ctx &c, const NttBatch &b, bool inv) {
    if (b.count <= 0) return;
    const int logN = c.log_n;
    if (c.n <= 32) {
        ntt_tiny_kernel<<<nblocks(b.count, 64), 64, 0, c.stream>>>(b, logN, inv ? 1 : 0, c.primes, inv ? c.itw : c.tw,
                                                                  inv ? c.itw_sh : c.tw_sh, c.ntt_const);
        check_launch("ntt_tiny_kernel");
        return;
    }
    if (c.n < 2048) {
        PassArgs a{logN, 0, logN, 1, 1, 1};
        if (inv) launch_pass<true, false>(c, b, a);
        else launch_pass<false, false>(c, b, a);
        return;
    }
    const int la = logN / 2, lb = logN - la;
    PassArgs p1{logN, 0, la, 16, 0, 0};
    PassArgs p2{logN, la, logN, (2048 >> lb) > 1 ? (2048 >> lb) : 1, 0, 0};
    if (!inv) {
        p1.first = 1;
        p2.last = 1;
        launch_pass<false, true>(c, b, p1);
        launch_pass<false, false>(c, b, p2);
    } else {
        p2.first = 1;
        p1.last = 1;
        launch_pass<true, false>(c, b, p2);
        launch_pass<true, true>(c, b, p1);
    }
}

}  // namespace

void ntt_forward(Ctx &c, const NttBatch &b) { run(c, b, false); }
void ntt_inverse(Ctx &c, const NttBatch &b) { run(c, b, true); }

}  // namespace vr
