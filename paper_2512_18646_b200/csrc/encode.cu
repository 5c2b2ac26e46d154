// encode.cu -- CKKS encode (canonical embedding), public/secret-key
// encryption, decryption + decode, and key generation, all on the device.
//
// Encode/decode is a length-S complex FFT (S = N/2) twisted by zeta^k
// (zeta = exp(i*pi/N)); slot j sits at DFT bin r_j = (5^j mod 2N - 1)/4, so the
// Galois map X -> X^(5^l) is a LEFT rotation by l, matching np.roll(-l) in
// engine.py:232-236.  Every floating-point operation uses explicit _rn
// intrinsics in the same order as oracle/ckks_oracle.c (compiled with
// -ffp-contract=off), so encoded integers are bit-identical to the oracle's.
//
// Randomness comes from the counter-based generator in modarith.cuh keyed by
// (seed, domain, nonce/digit, limb): identical integers on CPU and GPU, so
// ciphertext residues are bit-identical too.
#include "encode.cuh"

#include <vector>
#include "ntt_impl.cuh"

#include <cooperative_groups.h>

namespace vr {

namespace {

constexpr int TB = 256;

// Discrete Gaussian by CDT inversion: mag = #{i < CDT_LEN - 1 : r >= cdt[i]} (the table is
// non-decreasing), i.e. exactly the oracle's linear scan, found by a branch-free 5-step binary
// search -- no data-dependent loop, so a warp no longer waits for its largest sample.
__device__ __forceinline__ int64_t gauss(uint64_t u, const uint64_t *cdt) {
    static_assert(CDT_LEN == 32, "binary search covers 31 entries");
    const uint64_t r = u >> 1;
    int mag = 0;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1)
        if (r >= cdt[mag + s - 1]) mag += s;
    return (u & 1) ? -(int64_t)mag : (int64_t)mag;
}

__device__ __forceinline__ unsigned brev_bits(unsigned x, int bits) { return bits ? __brev(x) >> (32 - bits) : 0; }

// Slot FFT: radix-2 DIT over re/im (bit-reversed input already in place), executed as
// rounds of up to three consecutive stages held in registers (one barrier per round).
// Every butterfly sees the same operands and twiddle as the stage-by-stage loop of
// oracle/ckks_oracle.c, so the results are bit-identical; only the schedule differs.
// Shared-memory copies pad one double per eight so the stride-8 first round is conflict-free.
template <bool PAD>
__device__ __forceinline__ int fidx(int i) {
    return PAD ? i + (i >> 3) : i;
}

// RB consecutive stages on one register group x[u] = element b + u * h (b = j0 mod h):
// stage st has half-length hs = h * 2^st, butterfly (u, u + 2^st) uses twiddle j = j0 + (u mod 2^st) * h
template <int RB>
__device__ __forceinline__ void fft_group(double *xr, double *xi, int h, int j0, const double2 *tw, bool inverse) {
    constexpr int R = 1 << RB;
#pragma unroll
    for (int st = 0; st < RB; st++) {
        const int hs = h << st;
#pragma unroll
        for (int qb = 0; qb < (1 << st); qb++) {
            const double2 w = tw[hs + j0 + qb * h];
            const double wr = w.x, wi = inverse ? -w.y : w.y;
#pragma unroll
            for (int u = qb; u < R; u += 2 << st) {
                const int v = u + (1 << st);
                const double tr = __dsub_rn(__dmul_rn(xr[v], wr), __dmul_rn(xi[v], wi));
                const double ti = __dadd_rn(__dmul_rn(xr[v], wi), __dmul_rn(xi[v], wr));
                xr[v] = __dsub_rn(xr[u], tr);
                xi[v] = __dsub_rn(xi[u], ti);
                xr[u] = __dadd_rn(xr[u], tr);
                xi[u] = __dadd_rn(xi[u], ti);
            }
        }
    }
}

// stages with half-lengths h, 2h, .., h * 2^(RB-1) over an S-element block in (padded) shared memory
template <int RB>
__device__ __forceinline__ void fft_round(double *re, double *im, int S, int h, const double2 *tw, bool inverse) {
    constexpr int R = 1 << RB;
    const int G = S >> RB;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        const int j0 = g & (h - 1);
        const int b = (g - j0) * R + j0;
        double xr[R], xi[R];
#pragma unroll
        for (int u = 0; u < R; u++) {
            xr[u] = re[fidx<true>(b + u * h)];
            xi[u] = im[fidx<true>(b + u * h)];
        }
        fft_group<RB>(xr, xi, h, j0, tw, inverse);
#pragma unroll
        for (int u = 0; u < R; u++) {
            re[fidx<true>(b + u * h)] = xr[u];
            im[fidx<true>(b + u * h)] = xi[u];
        }
    }
}

// all stages of length 2 .. S (S = 2^logS), one barrier per round of up to three stages
// RBMAX = 2: radix-4 rounds (twice the threads per round, half the dependent chain per thread) for
// the latency-bound single-ciphertext decode; the butterflies and their order are unchanged.
// tws: shared-memory copy of the table's first `staged` entries (a round with half-length h and RB
// stages reads indices < h 2^RB); rounds reaching beyond it read the global table tw (L1-resident:
// every CTA of the launch reads the same entries).
template <int RBMAX = 3>
__device__ __forceinline__ void fft_stages(double *re, double *im, int S, int logS, const double2 *tw, const double2 *tws,
                                           int staged, bool inverse) {
    int h = 1, rem = logS;
    for (; rem >= RBMAX; rem -= RBMAX, h <<= RBMAX) {
        fft_round<RBMAX>(re, im, S, h, (h << RBMAX) <= staged ? tws : tw, inverse);
        __syncthreads();
    }
    if (rem == 2) {
        fft_round<2>(re, im, S, h, (h << 2) <= staged ? tws : tw, inverse);
        __syncthreads();
    } else if (rem == 1) {
        fft_round<1>(re, im, S, h, (h << 1) <= staged ? tws : tw, inverse);
        __syncthreads();
    }
}

// Slot-value source of ciphertext c: value(c, j) = src[c*sc + (j / p)*s1 + (j % p)*s2] for j < nvals.
// Dense rows: p = nvals, s1 = 0, s2 = 1, sc = nvals.  encode_left (slot i*p+j = A[i][c]): sc = 1,
// s1 = n, s2 = 0.  encode_right (slot i*p+j = B[c][j]): sc = p, s1 = 0, s2 = 1.  Image columns
// (slot b*h+i = img[b][i][c]): p = h, sc = 1, s1 = h*w, s2 = w.  Only the raw source crosses PCIe.
struct SlotSrc {
    const double *src;
    long long sc, s1, s2;
    int p, nvals;
    // optional second source for ciphertexts c >= split (two strided operands encrypted in one launch)
    const double *src_b = nullptr;
    long long sc_b = 0, s1_b = 0, s2_b = 0;
    int p_b = 1, nvals_b = 0, split = 0x7fffffff;
    __device__ __forceinline__ double at(int c, int j) const {
        if (c >= split) {
            if (j >= nvals_b) return 0.0;
            const int a = j / p_b, b = j - a * p_b;
            return src_b[(long long)(c - split) * sc_b + (long long)a * s1_b + (long long)b * s2_b];
        }
        if (j >= nvals) return 0.0;
        const int a = j / p, b = j - a * p;
        return src[(long long)c * sc + (long long)a * s1 + (long long)b * s2];
    }
};

// The FFT of one ciphertext is split over a cluster of CL CTAs: CTA r holds positions
// [r C, (r + 1) C) (C = S / CL) of the bit-reversed array in padded shared memory.  The
// first log2(C) stages are local; the last log2(CL) = 3 stages form one radix-8 round whose
// groups {j0 + u C} take element u from CTA u through distributed shared memory.
constexpr int FFT_CL = 8;

// The local stages read their twiddles (indices < C) from a shared-memory copy of the table's
// first C entries (tws, filled by stage_twiddles before the PDL wait: the table is constant, so
// its load overlaps the previous kernel); only the cross-cluster round reads the global table.
__device__ __forceinline__ void stage_twiddles(double2 *tws, const double2 *tw, int staged) {
    for (int i = threadIdx.x; i < staged; i += blockDim.x) tws[i] = __ldg(tw + i);
}
// Twiddles staged per CTA: the entries the full-radix local rounds read, 2^(RBMAX floor(log2 C / RBMAX)).
// A trailing partial round reads the global table, which keeps a 1024-point CTA at 26.6 KB of shared
// memory: eight CTAs per SM, so the 1024 CTAs of a 128-ciphertext cfg-2 encryption are one wave.
__host__ __device__ inline int fft_staged(int C, int rbmax) {
    int logc = 0;
    while ((1 << (logc + 1)) <= C) logc++;
    return 1 << (rbmax * (logc / rbmax));
}

template <int CL, int RBMAX = 3>
__device__ __forceinline__ void fft_cluster(double *re, double *im, int S, int logS, const double2 *tw, const double2 *tws,
                                            bool inverse) {
    const int C = S / CL;
    fft_stages<RBMAX>(re, im, C, logS - (CL == 8 ? 3 : 0), tw, tws, fft_staged(C, 3), inverse);
    if constexpr (CL == 8) {
        namespace cg = cooperative_groups;
        cg::cluster_group cluster = cg::this_cluster();
        cluster.sync();
        const int r = (int)cluster.block_rank(), per = C / 8;
        for (int g = threadIdx.x; g < per; g += blockDim.x) {
            const int j0 = r * per + g, jj = fidx<true>(j0);
            double xr[8], xi[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                xr[u] = cluster.map_shared_rank(re, u)[jj];
                xi[u] = cluster.map_shared_rank(im, u)[jj];
            }
            fft_group<3>(xr, xi, C, j0, tw, inverse);
#pragma unroll
            for (int u = 0; u < 8; u++) {
                cluster.map_shared_rank(re, u)[jj] = xr[u];
                cluster.map_shared_rank(im, u)[jj] = xi[u];
            }
        }
        cluster.sync();
    }
}

// Optional fused encryption noise (secret-key path): m += e with e the ciphertext's Gaussian
// sample (DOM_ENC_E0), so the NTT that follows only reduces m + e into each limb; the
// stream keys of the uniform a-polynomials are written to keys[c * nl + i].
struct EncNoise {
    const uint64_t *cdt;
    uint64_t seed, nonce0;
    int nl;
    uint64_t *keys;  // null: no noise
};

// cluster of CL CTAs per ciphertext: slot values -> m [count][N] (int64)
template <int CL, int RBMAX = 3>
__global__ void __launch_bounds__(512, 2) k_encode(SlotSrc vs, int S, int logS, double f, const double *zr, const double *zi, const double2 *tw,
                         const int *pos_slot, EncNoise nz, int64_t *m) {
    extern __shared__ double fft_sm[];
    __shared__ uint64_t cdt_s[CDT_LEN];
    const int C = S / CL, rank = (int)(blockIdx.x % CL), base = rank * C;
    const int c = blockIdx.x / CL;
    double *re = fft_sm, *im = fft_sm + C + C / 8;
    double2 *tws = reinterpret_cast<double2 *>(im + C + C / 8);
    stage_twiddles(tws, tw, fft_staged(C, 3));
    pdl_wait();
    pdl_trigger();
    if (nz.keys) {
        if (threadIdx.x < CDT_LEN) cdt_s[threadIdx.x] = nz.cdt[threadIdx.x];
        if (rank == 0 && threadIdx.x < nz.nl)
            nz.keys[(size_t)c * nz.nl + threadIdx.x] = stream_key(nz.seed, DOM_ENC_A, nz.nonce0 + (uint64_t)c, threadIdx.x);
    }
#pragma unroll 4
    for (int p = threadIdx.x; p < C; p += blockDim.x) {
        re[fidx<true>(p)] = vs.at(c, pos_slot[base + p]);
        im[fidx<true>(p)] = 0.0;
    }
    __syncthreads();
    fft_cluster<CL, RBMAX>(re, im, S, logS, tw, tws, true);
    int64_t *out = m + (size_t)c * 2 * S;
    const uint64_t ke = nz.keys ? stream_key(nz.seed, DOM_ENC_E0, nz.nonce0 + (uint64_t)c, 0) : 0;
#pragma unroll 4
    for (int p = threadIdx.x; p < C; p += blockDim.x) {
        const int k = base + p;
        const double yr = re[fidx<true>(p)], yi = im[fidx<true>(p)];
        const double xr = __dadd_rn(__dmul_rn(yr, zr[k]), __dmul_rn(yi, zi[k]));
        const double xi = __dsub_rn(__dmul_rn(yi, zr[k]), __dmul_rn(yr, zi[k]));
        int64_t v0 = __double2ll_rn(__dmul_rn(xr, f)), v1 = __double2ll_rn(__dmul_rn(xi, f));
        if (nz.keys) {
            v0 += gauss(rnd(ke, (uint64_t)k), cdt_s);
            v1 += gauss(rnd(ke, (uint64_t)(k + S)), cdt_s);
        }
        out[k] = v0;
        out[k + S] = v1;
    }
}

// cluster of CL CTAs per ciphertext: centred m [count][N], scales[count] -> real slots [count][S]
template <int CL, int RBMAX = 3>
__global__ void k_decode(const int64_t *m, const double *scales, int S, int logS, const double *zr, const double *zi,
                         const double2 *tw, const int *slot_pos, double *out) {
    extern __shared__ double fft_sm[];
    const int C = S / CL, rank = (int)(blockIdx.x % CL), base = rank * C;
    const int c = blockIdx.x / CL;
    double *re = fft_sm, *im = fft_sm + C + C / 8;
    double2 *tws = reinterpret_cast<double2 *>(im + C + C / 8);
    stage_twiddles(tws, tw, fft_staged(C, 3));
    if constexpr (RBMAX == 2) {
        // latency-bound single-ciphertext decode: the constant twist tables zr/zi (read at bit-reversed
        // positions spread over every line) and this CTA's slot map go to L2 before the PDL wait
        const int lines = S / 16;  // 128-byte lines of one [S] double table
        for (int l = rank * (lines / CL) + threadIdx.x; l < (rank + 1) * (lines / CL); l += blockDim.x) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(zr + 16 * l));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(zi + 16 * l));
        }
        for (int l = threadIdx.x; l < C / 32; l += blockDim.x) asm volatile("prefetch.global.L2 [%0];" ::"l"(slot_pos + base + 32 * l));
    }
    pdl_wait();
    pdl_trigger();
    const int64_t *mc = m + (size_t)c * 2 * S;
    const double scale = scales[c];
#pragma unroll 4
    for (int p = threadIdx.x; p < C; p += blockDim.x) {
        const int k = (int)brev_bits((unsigned)(base + p), logS);
        const double ur = __ddiv_rn(__ll2double_rn(mc[k]), scale), ui = __ddiv_rn(__ll2double_rn(mc[k + S]), scale);
        re[fidx<true>(p)] = __dsub_rn(__dmul_rn(ur, zr[k]), __dmul_rn(ui, zi[k]));
        im[fidx<true>(p)] = __dadd_rn(__dmul_rn(ur, zi[k]), __dmul_rn(ui, zr[k]));
    }
    __syncthreads();
    fft_cluster<CL, RBMAX>(re, im, S, logS, tw, tws, false);
    double *o = out + (size_t)c * S;
    if constexpr (CL == 8) {
        namespace cg = cooperative_groups;
        cg::cluster_group cluster = cg::this_cluster();
#pragma unroll 4
        for (int p = threadIdx.x; p < C; p += blockDim.x) {
            const int pos = slot_pos[base + p];  // C = 2^(logS - 3)
            o[base + p] = cluster.map_shared_rank(re, pos >> (logS - 3))[fidx<true>(pos & (C - 1))];
        }
        cluster.sync();  // peers keep their shared memory until every gather has finished
    } else {
        for (int p = threadIdx.x; p < C; p += blockDim.x) o[p] = re[fidx<true>(slot_pos[p])];
    }
}

// m [count][N] (int64) -> residues [count][nl][N] (coefficient domain)
__global__ void k_reduce_coeffs(const int64_t *m, int count, int nl, int N, DevPrimes pr, uint64_t *out) {
    pdl_wait();
    pdl_trigger();
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)count * nl * N) return;
    const int k = (int)(e % N);
    const long long ci = e / N;
    const int i = (int)(ci % nl);
    const long long c = ci / nl;
    out[e] = from_i64(m[c * N + k], pr.m[i]);
}

// public-key encryption samples: buf [count][3][nl][N] = (v, m + e0, e1) per limb
// secret-key encryption:          buf [count][2][nl][N] = (m + e, a (already NTT))
__global__ void k_enc_sample(const int64_t *m, int count, int nl, int N, uint64_t seed, uint64_t nonce0, int sym,
                             const uint64_t *cdt, DevPrimes pr, uint64_t *buf) {
    pdl_wait();
    pdl_trigger();
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)count * N) return;
    const long long c = e / N;
    const int k = (int)(e - c * N);
    const uint64_t nonce = nonce0 + (uint64_t)c;
    const int64_t e0 = gauss(rnd(stream_key(seed, DOM_ENC_E0, nonce, 0), k), cdt) + m[e];
    if (sym) {
        uint64_t *b = buf + (size_t)c * 2 * nl * N;
        for (int i = 0; i < nl; i++) {
            b[(size_t)i * N + k] = from_i64(e0, pr.m[i]);
            b[(size_t)(nl + i) * N + k] = sample_uniform(rnd(stream_key(seed, DOM_ENC_A, nonce, i), k), pr.m[i].q);
        }
        return;
    }
    const int64_t v = sample_ternary(rnd(stream_key(seed, DOM_ENC_V, nonce, 0), k));
    const int64_t e1 = gauss(rnd(stream_key(seed, DOM_ENC_E1, nonce, 0), k), cdt);
    uint64_t *b = buf + (size_t)c * 3 * nl * N;
    for (int i = 0; i < nl; i++) {
        b[(size_t)i * N + k] = from_i64(v, pr.m[i]);
        b[(size_t)(nl + i) * N + k] = from_i64(e0, pr.m[i]);
        b[(size_t)(2 * nl + i) * N + k] = from_i64(e1, pr.m[i]);
    }
}

// combine NTT'd samples into ciphertexts out [count][2][nl][N]
__global__ void k_enc_combine(const uint64_t *buf, int count, int nl, int N, int Ltop, int sym, const uint64_t *pk,
                              const uint64_t *s_ntt, DevPrimes pr, uint64_t *out) {
    pdl_wait();
    pdl_trigger();
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)count * nl * N) return;
    const int k = (int)(e % N);
    const long long ci = e / N;
    const int i = (int)(ci % nl);
    const long long c = ci / nl;
    const Modulus m = pr.m[i];
    uint64_t *o = out + (size_t)c * 2 * nl * N;
    if (sym) {
        const uint64_t *b = buf + (size_t)c * 2 * nl * N;
        const uint64_t me = b[(size_t)i * N + k], a = b[(size_t)(nl + i) * N + k];
        o[(size_t)i * N + k] = sub_mod(me, mul_mod(a, s_ntt[(size_t)i * N + k], m), m.q);
        o[(size_t)(nl + i) * N + k] = a;
        return;
    }
    const uint64_t *b = buf + (size_t)c * 3 * nl * N;
    const uint64_t v = b[(size_t)i * N + k], me0 = b[(size_t)(nl + i) * N + k], e1 = b[(size_t)(2 * nl + i) * N + k];
    const uint64_t p0 = pk[(size_t)i * N + k], p1 = pk[(size_t)(Ltop + 1 + i) * N + k];
    o[(size_t)i * N + k] = add_mod(mul_mod(v, p0, m), me0, m.q);
    o[(size_t)(nl + i) * N + k] = add_mod(mul_mod(v, p1, m), e1, m.q);
}

// ---- key generation ----
__global__ void k_sample_secret(int n, int np, uint64_t seed, DevPrimes pr, uint64_t *s) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)np * n) return;
    const int p = (int)(e / n), k = (int)(e - (long long)p * n);
    const int64_t v = sample_ternary(rnd(stream_key(seed, DOM_SK, 0, 0), k));
    s[e] = from_i64(v, pr.m[p]);
}

// pk: a_i uniform (NTT domain), e gaussian (coeff) -> buf_e [nl][N]
__global__ void k_pk_sample(int n, int nl, uint64_t seed, const uint64_t *cdt, DevPrimes pr, uint64_t *pk_a, uint64_t *e_buf) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)nl * n) return;
    const int i = (int)(e / n), k = (int)(e - (long long)i * n);
    pk_a[e] = sample_uniform(rnd(stream_key(seed, DOM_PK_A, 0, i), k), pr.m[i].q);
    e_buf[e] = from_i64(gauss(rnd(stream_key(seed, DOM_PK_E, 0, 0), k), cdt), pr.m[i]);
}

__global__ void k_pk_combine(int n, int nl, const uint64_t *s_ntt, const uint64_t *e_ntt, DevPrimes pr, uint64_t *pk) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)nl * n) return;
    const int i = (int)(e / n);
    const Modulus m = pr.m[i];
    const uint64_t a = pk[(size_t)nl * n + e];
    pk[e] = add_mod(neg_mod(mul_mod(a, s_ntt[e], m), m.q), e_ntt[e], m.q);
}

// switching key for s' (NTT, [np][N]): key [L+1][2][np][N]; e_buf [L+1][np][N]
__global__ void k_gkey_sample(int n, int nd, int np, uint64_t seed, uint64_t dom_a, uint64_t dom_e, uint64_t id,
                              const uint64_t *cdt, DevPrimes pr, uint64_t *key, uint64_t *e_buf) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)nd * np * n) return;
    const int k = (int)(e % n);
    const long long jp = e / n;
    const int p = (int)(jp % np), j = (int)(jp / np);
    key[(((size_t)j * 2 + 1) * np + p) * n + k] =
        sample_uniform(rnd(stream_key(seed, dom_a, id, (uint64_t)j * 256 + p), k), pr.m[p].q);
    e_buf[e] = from_i64(gauss(rnd(stream_key(seed, dom_e, id, j), k), cdt), pr.m[p]);
}

__global__ void k_gkey_combine(int n, int nd, int np, const uint64_t *s_ntt, const uint64_t *sp_ntt, const uint64_t *e_ntt,
                               DevPrimes pr, uint64_t *key) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)nd * np * n) return;
    const int k = (int)(e % n);
    const long long jp = e / n;
    const int p = (int)(jp % np), j = (int)(jp / np);
    const Modulus m = pr.m[p];
    const size_t pk_ = (size_t)p * n + k;
    const uint64_t a = key[(((size_t)j * 2 + 1) * np + p) * n + k];
    uint64_t v = add_mod(neg_mod(mul_mod(a, s_ntt[pk_], m), m.q), e_ntt[e], m.q);
    if (p == j) {
        const uint64_t pm = reduce64(pr.m[np - 1].q, m);
        v = add_mod(v, mul_mod(pm, sp_ntt[pk_], m), m.q);
    }
    key[(((size_t)j * 2 + 0) * np + p) * n + k] = v;
}

__global__ void k_square(const uint64_t *s, int np, int n, DevPrimes pr, uint64_t *out) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)np * n) return;
    const int p = (int)(e / n);
    out[e] = mul_mod(s[e], s[e], pr.m[p]);
}

__global__ void k_perm_rows(const uint64_t *in, int rows, int logN, uint32_t g, uint64_t *out) {
    const int N = 1 << logN;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)rows * N) return;
    const int k = (int)(e & (N - 1));
    const uint32_t brk = __brev((uint32_t)k) >> (32 - logN);
    const uint32_t ex = ((2u * brk + 1u) * g) & ((2u << logN) - 1u);
    const int src = (int)(__brev((ex - 1u) >> 1) >> (32 - logN));
    out[e] = in[(e - k) + src];
}

// Fused secret-key encryption: the NTT of (m + e) mod q_i reads its input straight from the
// sampler, and its store writes c0 = NTT(m + e) - a s and c1 = a (a sampled in the NTT domain).
// secret-key encryption through one fused forward NTT: load m + e (noise added by k_encode),
// store c0 = (m + e) - a * s and c1 = a with a uniform from the per-transform stream key
// On an FP64-body prime any |m + e| < 2^47 enters the transform unreduced, shifted by
// kshift[p] = q ceil(2^47 / q) (== 0 mod q) into [0, 2^48 + q); larger values are reduced.
struct LdSymEnc {
    const int64_t *m;
    int nl, N;
    uint64_t f64mask;
    const uint64_t *kshift;
    struct Prep {
        const int64_t *m;
        int64_t ks;  // < 0: the integer body (always reduce)
        Modulus mod;
    };
    __device__ __forceinline__ Prep prep(int t, const DevPrimes &pr, int pidx) const {
        Prep p;
        p.m = m + (long long)(t / nl) * N;
        p.ks = ((f64mask >> pidx) & 1ull) ? (int64_t)kshift[pidx] : -1;
        p.mod = pr.m[pidx];
        return p;
    }
    __device__ __forceinline__ uint64_t load(const Prep &p, long long E) const {
        const int64_t v = p.m[E];
        if (p.ks >= 0 && v > -(1ll << 47) && v < (1ll << 47)) return (uint64_t)(v + p.ks);
        return from_i64(v, p.mod);
    }
};
struct StSymEnc {
    const uint64_t *s_ntt, *s_sh, *keys;
    int nl, N;
    struct Pre {
        uint64_t s, s_sh;
    };
    struct Ctx {
        const uint64_t *s, *s_sh;
        uint64_t *c0;
        uint64_t key, q;
        long long c1_off;
    };
    __device__ __forceinline__ Ctx ctx(uint64_t *ptr, int t, const DevPrimes &pr, int pidx) const {
        const long long o = (long long)(t % nl) * N;
        return Ctx{s_ntt + o, s_sh + o, ptr, keys[t], pr.m[pidx].q, (long long)nl * N};
    }
    __device__ __forceinline__ Pre prefetch(const Ctx &c, long long E) const { return Pre{c.s[E], c.s_sh[E]}; }
    __device__ __forceinline__ void finish(const Ctx &c, long long E, uint64_t v, const Pre &p) const {
        const uint64_t a = sample_uniform(rnd(c.key, (uint64_t)E), c.q);
        c.c0[E] = sub_mod(v, mul_shoup(a, p.s, p.s_sh, c.q), c.q);
        c.c0[c.c1_off + E] = a;
    }
};

int log2i(int x) {
    int l = 0;
    while ((1 << l) < x) l++;
    return l;
}

int fft_cl(int S) { return S >= 64 ? FFT_CL : 1; }
int fft_threads(int S) {
    const int C = S / fft_cl(S);
    return C >= 2048 ? 256 : (C >= 256 ? C / 8 : 32);
}
size_t fft_smem(int S) {
    const int C = S / fft_cl(S);
    return (size_t)2 * (C + C / 8) * sizeof(double) + (size_t)fft_staged(C, 3) * sizeof(double2);  // re, im (padded) + twiddles
}

template <typename K, typename... Args>
void launch_fft_t(Ctx &c, K kern, int count, int S, int tmul, Args... args) {
    const int cl = fft_cl(S);
    const size_t sm = fft_smem(S);
    ensure_smem(c, (const void *)kern, sm);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(count * cl));
    cfg.blockDim = dim3((unsigned)(fft_threads(S) * tmul));
    cfg.dynamicSmemBytes = sm;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[3];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = add_priority_attr(attr, pdl_enabled() ? 2 : 1);
    VR_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

template <typename K, typename... Args>
void launch_fft(Ctx &c, K kern, int count, int S, Args... args) {
    launch_fft_t(c, kern, count, S, 1, args...);
}

}  // namespace

static void encode_src(Ctx &c, const SlotSrc &vs, int count, double scale, int64_t *d_m, EncNoise nz = EncNoise{}) {
    const int S = c.slots;
    const double f = scale / (double)S;
    const double2 *tw = reinterpret_cast<const double2 *>(c.ftw);
    if (count <= 0) return;
    // VR_ENC_R4=1: radix-4 rounds with twice the threads (measured slower for the 64-ciphertext
    // batches of cfg 2: 24 -> 30.5 us; the decode of <= 4 ciphertexts uses them, 25 -> 17 us)
    static const int enc_r4 = [] {
        const char *e = getenv("VR_ENC_R4");
        return e ? atoi(e) : 0;
    }();
    if (fft_cl(S) == FFT_CL) {
        if (enc_r4 && fft_threads(S) <= 512)
            launch_fft_t(c, k_encode<FFT_CL, 2>, count, S, 2, vs, S, log2i(S), f, (const double *)c.zr, (const double *)c.zi,
                         tw, (const int *)c.pos_slot, nz, d_m);
        else
            launch_fft(c, k_encode<FFT_CL>, count, S, vs, S, log2i(S), f, (const double *)c.zr, (const double *)c.zi, tw,
                       (const int *)c.pos_slot, nz, d_m);
    } else {
        launch_fft(c, k_encode<1>, count, S, vs, S, log2i(S), f, (const double *)c.zr, (const double *)c.zi, tw,
                   (const int *)c.pos_slot, nz, d_m);
    }
    check_launch("k_encode");
}

void encode_coeffs(Ctx &c, const double *d_vals, int count, int nvals, double scale, int64_t *d_m) {
    encode_src(c, SlotSrc{d_vals, nvals, 0, 1, nvals > 0 ? nvals : 1, nvals}, count, scale, d_m);
}

void encode_plain(Ctx &c, const double *d_vals, int count, int nvals, int level, double scale, uint64_t *d_pt) {
    const int N = c.n, nl = level + 1;
    Scratch m(c, sizeof(int64_t) * count * N);
    encode_coeffs(c, d_vals, count, nvals, scale, m.as<int64_t>());
    launch_pdl(k_reduce_coeffs, dim3(nblocks((long long)count * nl * N, TB)), dim3(TB), 0, c.stream, m.as<int64_t>(), count, nl, N, c.primes, d_pt);
    check_launch("k_reduce_coeffs");
    ntt_forward(c, batch_limbs(d_pt, count, nl, N));
}

void encrypt_src(Ctx &c, const double *src, long long sc, long long s1, long long s2, int p, int nvals, int count, int level,
                 double scale, uint64_t nonce0, uint64_t *d_ct);

void encrypt(Ctx &c, const double *d_vals, int count, int nvals, int level, double scale, uint64_t nonce0, uint64_t *d_ct) {
    encrypt_src(c, d_vals, nvals, 0, 1, nvals > 0 ? nvals : 1, nvals, count, level, scale, nonce0, d_ct);
}

// Two strided operands (encode_left + encode_right of one product) as ONE secret-key encryption: one
// slot-FFT launch and one fused NTT over both batches (ciphertexts count0.. go to d_ct2, nonces stay
// consecutive), so the latency-bound encode and the NTT's tail are paid once.
void encrypt_src2(Ctx &c, const double *src0, long long sc0, long long s1_0, long long s2_0, int p0, int nvals0, int count0,
                  uint64_t *d_ct0, const double *src1, long long sc1, long long s1_1, long long s2_1, int p1, int nvals1,
                  int count1, uint64_t *d_ct1, int level, double scale, uint64_t nonce0) {
    if (!c.sym_enc) throw VrError(3, "combined encryption needs secret-key encryption");
    c.enc_calls++;
    const int N = c.n, nl = level + 1, count = count0 + count1;
    Scratch m(c, sizeof(int64_t) * count * N), keys(c, sizeof(uint64_t) * count * nl);
    SlotSrc vs{src0, sc0, s1_0, s2_0, p0 > 0 ? p0 : 1, nvals0};
    vs.src_b = src1;
    vs.sc_b = sc1;
    vs.s1_b = s1_1;
    vs.s2_b = s2_1;
    vs.p_b = p1 > 0 ? p1 : 1;
    vs.nvals_b = nvals1;
    vs.split = count0;
    encode_src(c, vs, count, scale, m.as<int64_t>(), EncNoise{c.cdt, c.seed, nonce0, nl, keys.as<uint64_t>()});
    NttBatch b{d_ct0, count * nl, nl, (long long)2 * nl * N, nl, 0, 0, 0};
    b.data2 = d_ct1;
    b.split = count0 * nl;
    ntt_forward_fused(c, b, LdSymEnc{m.as<int64_t>(), nl, N, c.f64mask, c.kshift},
                      StSymEnc{c.s_ntt, c.s_sh, keys.as<uint64_t>(), nl, N});
}

void encrypt_src(Ctx &c, const double *src, long long sc, long long s1, long long s2, int p, int nvals, int count, int level,
                 double scale, uint64_t nonce0, uint64_t *d_ct) {
    const int N = c.n, nl = level + 1;
    c.enc_calls++;
    Scratch m(c, sizeof(int64_t) * count * N);
    const SlotSrc vs{src, sc, s1, s2, p > 0 ? p : 1, nvals};
    if (c.sym_enc) {
        // encode adds e; one fused NTT (2 passes): m + e -> NTT -> (c0, c1), in place in the output ciphertexts
        Scratch keys(c, sizeof(uint64_t) * count * nl);
        encode_src(c, vs, count, scale, m.as<int64_t>(), EncNoise{c.cdt, c.seed, nonce0, nl, keys.as<uint64_t>()});
        ntt_forward_fused(c, NttBatch{d_ct, count * nl, nl, (long long)2 * nl * N, nl, 0, 0, 0},
                          LdSymEnc{m.as<int64_t>(), nl, N, c.f64mask, c.kshift}, StSymEnc{c.s_ntt, c.s_sh, keys.as<uint64_t>(), nl, N});
        return;
    }
    encode_src(c, vs, count, scale, m.as<int64_t>());
    const int rows = c.sym_enc ? 2 : 3;
    Scratch buf(c, sizeof(uint64_t) * count * rows * nl * N);
    launch_pdl(k_enc_sample, dim3(nblocks((long long)count * N, TB)), dim3(TB), 0, c.stream, m.as<int64_t>(), count, nl, N, c.seed, nonce0,
                                                                         c.sym_enc, c.cdt, c.primes, buf.as<uint64_t>());
    check_launch("k_enc_sample");
    if (c.sym_enc) {
        // only the (m + e) rows need a forward NTT: rows at [c][0][*]
        ntt_forward(c, NttBatch{buf.as<uint64_t>(), count * nl, nl, (long long)2 * nl * N, nl, 0, 0, 0});
    } else {
        ntt_forward(c, batch_limbs(buf.as<uint64_t>(), count * 3, nl, N));
    }
    launch_pdl(k_enc_combine, dim3(nblocks((long long)count * nl * N, TB)), dim3(TB), 0, c.stream, buf.as<uint64_t>(), count, nl, N, c.L,
                                                                               c.sym_enc, c.pk, c.s_ntt, c.primes, d_ct);
    check_launch("k_enc_combine");
}

// decryption fused into the limb-0 inverse NTT: the load computes c0 + c1 s (+ c2 s^2) mod q0 in the
// NTT domain, the store centres the coefficients into int64
struct LdDec {
    const uint64_t *const *C;
    const int *degs, *levels;
    const uint64_t *s_ntt;
    int N;
    __device__ __forceinline__ uint64_t operator()(const uint64_t *, int t, long long E, const DevPrimes &pr, int) const {
        const Modulus m = pr.m[0];
        const uint64_t *ct = C[t];
        const long long nlN = (long long)(levels[t] + 1) * N;
        const uint64_t s = s_ntt[E];
        uint64_t v = add_mod(ct[E], mul_mod(ct[nlN + E], s, m), m.q);
        if (degs[t] == 2) v = add_mod(v, mul_mod(ct[2 * nlN + E], mul_mod(s, s, m), m), m.q);
        return v;
    }
};
struct StCenter {
    int64_t *m;
    uint64_t q;
    int N;
    struct Pre {};
    __device__ __forceinline__ Pre prefetch(int, long long, const DevPrimes &, int) const { return Pre{}; }
    __device__ __forceinline__ void finish(uint64_t *, int t, long long E, uint64_t v, const Pre &, const DevPrimes &, int) const {
        m[(long long)t * N + E] = v > (q >> 1) ? -(int64_t)(q - v) : (int64_t)v;
    }
};

void decrypt_decode(Ctx &c, const uint64_t *const *d_cts, const int *d_degs, const int *d_levels, const double *d_scales,
                    int count, double *d_out, int64_t *d_coeffs_out) {
    const int N = c.n, S = c.slots;
    Scratch x(c, sizeof(uint64_t) * count * N), m(c, sizeof(int64_t) * count * N);
    int64_t *mp = d_coeffs_out ? d_coeffs_out : m.as<int64_t>();
    ntt_inverse_fused(c, NttBatch{x.as<uint64_t>(), count, 1, (long long)N, 1, 0, 0, 0},
                      LdDec{d_cts, d_degs, d_levels, c.s_ntt, N}, StCenter{mp, c.q[0], N});
    if (!d_out) return;
    const double2 *tw = reinterpret_cast<const double2 *>(c.ftw);
    if (count > 0) {
        if (fft_cl(S) == FFT_CL) {
            if (count <= 4 && fft_threads(S) <= 512)  // latency-bound: radix-4 rounds, twice the threads
                launch_fft_t(c, k_decode<FFT_CL, 2>, count, S, 2, (const int64_t *)mp, d_scales, S, log2i(S),
                             (const double *)c.zr, (const double *)c.zi, tw, (const int *)c.slot_pos, d_out);
            else
                launch_fft(c, k_decode<FFT_CL>, count, S, (const int64_t *)mp, d_scales, S, log2i(S), (const double *)c.zr,
                           (const double *)c.zi, tw, (const int *)c.slot_pos, d_out);
        } else
            launch_fft(c, k_decode<1>, count, S, (const int64_t *)mp, d_scales, S, log2i(S), (const double *)c.zr,
                       (const double *)c.zi, tw, (const int *)c.slot_pos, d_out);
    }
    check_launch("k_decode");
}

void keygen(Ctx &c) {
    const int n = c.n, np = c.np, nl = c.L + 1;
    VR_CUDA(cudaMallocAsync((void **)&c.s_ntt, sizeof(uint64_t) * np * n, c.stream));
    k_sample_secret<<<nblocks((long long)np * n, TB), TB, 0, c.stream>>>(n, np, c.seed, c.primes, c.s_ntt);
    check_launch("k_sample_secret");
    ntt_forward(c, batch_limbs(c.s_ntt, 1, np, n));
    {
        // Shoup companions of s (encryption multiplies every a-polynomial by s)
        std::vector<uint64_t> h((size_t)np * n);
        VR_CUDA(cudaMemcpyAsync(h.data(), c.s_ntt, sizeof(uint64_t) * h.size(), cudaMemcpyDeviceToHost, c.stream));
        VR_CUDA(cudaStreamSynchronize(c.stream));
        for (int i = 0; i < np; i++)
            for (int k = 0; k < n; k++) {
                uint64_t &v = h[(size_t)i * n + k];
                v = (uint64_t)(((unsigned __int128)v << 64) / c.q[i]);
            }
        VR_CUDA(cudaMalloc((void **)&c.s_sh, sizeof(uint64_t) * h.size()));
        VR_CUDA(cudaMemcpy(c.s_sh, h.data(), sizeof(uint64_t) * h.size(), cudaMemcpyHostToDevice));
    }
    VR_CUDA(cudaMallocAsync((void **)&c.pk, sizeof(uint64_t) * 2 * nl * n, c.stream));
    Scratch e(c, sizeof(uint64_t) * nl * n);
    k_pk_sample<<<nblocks((long long)nl * n, TB), TB, 0, c.stream>>>(n, nl, c.seed, c.cdt, c.primes, c.pk + (size_t)nl * n,
                                                                     e.as<uint64_t>());
    check_launch("k_pk_sample");
    ntt_forward(c, batch_limbs(e.as<uint64_t>(), 1, nl, n));
    k_pk_combine<<<nblocks((long long)nl * n, TB), TB, 0, c.stream>>>(n, nl, c.s_ntt, e.as<uint64_t>(), c.primes, c.pk);
    check_launch("k_pk_combine");
}

static uint64_t *gen_switch_key(Ctx &c, const uint64_t *sp_ntt, uint64_t dom_a, uint64_t dom_e, uint64_t id) {
    const int n = c.n, np = c.np, nd = c.L + 1;
    uint64_t *key = nullptr;
    VR_CUDA(cudaMalloc((void **)&key, sizeof(uint64_t) * c.key_words()));
    Scratch e(c, sizeof(uint64_t) * nd * np * n);
    const long long tot = (long long)nd * np * n;
    k_gkey_sample<<<nblocks(tot, TB), TB, 0, c.stream>>>(n, nd, np, c.seed, dom_a, dom_e, id, c.cdt, c.primes, key,
                                                         e.as<uint64_t>());
    check_launch("k_gkey_sample");
    ntt_forward(c, batch_limbs(e.as<uint64_t>(), nd, np, n));
    k_gkey_combine<<<nblocks(tot, TB), TB, 0, c.stream>>>(n, nd, np, c.s_ntt, sp_ntt, e.as<uint64_t>(), c.primes, key);
    check_launch("k_gkey_combine");
    return key;
}

uint64_t *relin_key(Ctx &c) {
    if (!c.rlk) {
        Scratch s2(c, sizeof(uint64_t) * c.np * c.n);
        k_square<<<nblocks((long long)c.np * c.n, TB), TB, 0, c.stream>>>(c.s_ntt, c.np, c.n, c.primes, s2.as<uint64_t>());
        check_launch("k_square");
        c.rlk = gen_switch_key(c, s2.as<uint64_t>(), DOM_RLK_A, DOM_RLK_E, 0);
    }
    return c.rlk;
}

uint64_t *galois_key(Ctx &c, uint32_t g) {
    auto it = c.gkeys.find(g);
    if (it != c.gkeys.end()) return it->second;
    Scratch sg(c, sizeof(uint64_t) * c.np * c.n);
    k_perm_rows<<<nblocks((long long)c.np * c.n, TB), TB, 0, c.stream>>>(c.s_ntt, c.np, c.log_n, g, sg.as<uint64_t>());
    check_launch("k_perm_rows");
    uint64_t *key = gen_switch_key(c, sg.as<uint64_t>(), DOM_GAL_A, DOM_GAL_E, g);
    c.gkeys[g] = key;
    return key;
}

}  // namespace vr
