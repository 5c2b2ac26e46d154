// keyswitch.cu -- rescale, hybrid key switching (ModUp -> inner product ->
// ModDown), relinearisation and hoisted Galois rotations.
//
// Key switching follows oracle/ckks_oracle.c:orc_keyswitch exactly: dnum = l+1
// single-prime digits d_j = [c]_{q_j} (centred), lifted to every q_t and the
// special prime P, NTT'd, multiplied with the key rows ([L+1][2][np][N]) and
// summed, then divided by P with rounding (ModDown).  Rotation by Galois
// element g permutes the already-ModUp'd digits on read, which is bit-exact
// with switching the permuted polynomial (lift and NTT commute with the
// signed coefficient permutation), so one ModUp serves every rotation amount.
//
// Kernel count per key switch: ModUp = INTT (gather prologue) + NTT (lift
// prologue); inner product; ModDown = INTT (strided prologue) + NTT (lift
// prologue, "(a - z) * P^-1 (+ add)" epilogue).  Each NTT is two passes.
#include <cstdlib>

#include "ntt_impl.cuh"
#include "ring.cuh"

namespace vr {

namespace {

constexpr int TB = 256;

__device__ __forceinline__ int galois_src(int k, uint32_t g, int logN) {
    if (g == 1) return k;
    const uint32_t brk = __brev((uint32_t)k) >> (32 - logN);
    const uint32_t e = ((2u * brk + 1u) * g) & ((2u << logN) - 1u);
    return (int)(__brev((e - 1u) >> 1) >> (32 - logN));
}

// base + t*stride + off + E
struct LdStrided {
    const uint64_t *base;
    long long stride, off;
    __device__ __forceinline__ uint64_t operator()(const uint64_t *, int t, long long E, const DevPrimes &, int) const {
        return base[(long long)t * stride + off + E];
    }
};

// A[c][x][t][k] = sum_j D[c][j][t][src(k)] * key[j][x][pidx(t)][k]; the digit's own
// prime (t == j) is read from the input polynomial (ModUp never materialises it).
// Grid (t*N + k, ciphertext groups of CG): a thread keeps its key column
// (2 x (l+1) words) in registers and issues all CG x (l+1) digit loads before
// the multiply-accumulates, so the key is read count/CG times per launch and
// every thread has CG*(l+1) independent loads in flight.
template <int KS_MAXD, int KS_CG>
__global__ void __launch_bounds__(128) k_ks_inner(const uint64_t *D, const uint64_t *const *P, long long poly_off, int count,
                                                  int level, int N, int logN, int np, const uint64_t *key, uint32_t g,
                                                  DevPrimes pr, uint64_t *A, const NttConst *__restrict__ ncs,
                                                  const uint64_t *const *keys_r, const uint32_t *gs_r) {
    // keys_r: one launch for every rotation amount of a hoisted batch (grid z = amount r): key and
    // Galois element of amount r, output ciphertext c*nrot + r
    const int nrot = gridDim.z, rz = blockIdx.z;
    if (keys_r) {
        key = keys_r[rz];
        g = gs_r[rz];
    }
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int nl = level + 1, nt = level + 2;
    if (e >= (long long)nt * N) {
        pdl_wait();
        pdl_trigger();
        return;
    }
    const int k = (int)(e % N), t = (int)(e / N);
    const int c0 = blockIdx.y * KS_CG;
    const int pidx = t < nl ? t : np - 1;
    const Modulus m = pr.m[pidx];
    const int src = galois_src(k, g, logN);
    // the key is constant: its loads are issued before the PDL wait (they overlap the ModUp tail)
    uint64_t k0[KS_MAXD], k1[KS_MAXD];
#pragma unroll
    for (int j = 0; j < KS_MAXD; j++) {
        if (j < nl) {
            k0[j] = __ldg(key + (((size_t)j * 2 + 0) * np + pidx) * N + k);
            k1[j] = __ldg(key + (((size_t)j * 2 + 1) * np + pidx) * N + k);
        }
    }
    pdl_wait();
    pdl_trigger();
    uint64_t dv[KS_CG][KS_MAXD];
#pragma unroll
    for (int cc = 0; cc < KS_CG; cc++) {
        const int c = c0 + cc;
        if (c >= count) break;
#pragma unroll
        for (int j = 0; j < KS_MAXD; j++)
            if (j < nl)
                dv[cc][j] = (t == j) ? P[c][poly_off + (long long)j * N + src] : D[(((long long)c * nl + j) * nt + t) * N + src];
    }
    const NttConst nc = ncs[pidx];
    if (nc.f64) {
        // FP64 pipe (prime < 2^46): exact Shoup-style products, sums of |r| <= q stay exact in a double
        double kd0[KS_MAXD], kd1[KS_MAXD];
#pragma unroll
        for (int j = 0; j < KS_MAXD; j++)
            if (j < nl) {
                kd0[j] = nttk::u2d(k0[j]);
                kd1[j] = nttk::u2d(k1[j]);
            }
#pragma unroll
        for (int cc = 0; cc < KS_CG; cc++) {
            const int c = c0 + cc;
            if (c >= count) break;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int j = 0; j < KS_MAXD; j++)
                if (j < nl) {
                    const double dd = nttk::u2d(dv[cc][j]);
                    a0 = __dadd_rn(a0, nttk::mulmod_f(dd, kd0[j], nc.qd, nc.qinv));
                    a1 = __dadd_rn(a1, nttk::mulmod_f(dd, kd1[j], nc.qd, nc.qinv));
                }
            const long long co = (long long)c * nrot + rz;
            A[((co * 2 + 0) * nt + t) * N + k] = nttk::canon_f(a0, nc.qd, nc.qinv);
            A[((co * 2 + 1) * nt + t) * N + k] = nttk::canon_f(a1, nc.qd, nc.qinv);
        }
        return;
    }
#pragma unroll
    for (int cc = 0; cc < KS_CG; cc++) {
        const int c = c0 + cc;
        if (c >= count) break;
        u128 a0{0, 0}, a1{0, 0};
#pragma unroll
        for (int j = 0; j < KS_MAXD; j++) {
            if (j < nl) {
                // no fold inside the sum: q < 2^61, so KS_MAXD <= 64 products below 2^122 fit 128 bits
                mac_to(a0, dv[cc][j], k0[j]);
                mac_to(a1, dv[cc][j], k1[j]);
            }
        }
        const long long co = (long long)c * nrot + rz;
        A[((co * 2 + 0) * nt + t) * N + k] = reduce128(a0, m);
        A[((co * 2 + 1) * nt + t) * N + k] = reduce128(a1, m);
    }
}

// ---- fused relinearise + rescale (oracle/ckks_oracle.c:orc_relin_rescale) ----------
// X_b = P * d_b + acc_b; rows of Y: 0 = X_b mod q_l, 1 = acc_b mod P (= X_b mod P)
struct LdXrow {
    const uint64_t *A;              // [count][2][nt][N] accumulators
    const uint64_t *const *D3;      // relin inputs [3][l+1][N]
    const uint64_t *rr;             // rr_tab row for this level
    int level, nt, N;
    __device__ __forceinline__ uint64_t operator()(const uint64_t *, int t, long long E, const DevPrimes &pr, int) const {
        const int cb = t >> 1, w = t & 1, c = cb >> 1, b = cb & 1;
        const uint64_t *a = A + ((long long)cb * nt) * N;
        if (w) return a[(long long)(nt - 1) * N + E];
        const uint64_t q = pr.m[level].q;
        const uint64_t d = D3[c][((long long)b * (level + 1) + level) * N + E];
        return add_mod(mul_shoup(d, rr[MAXP * 8 + 0], rr[MAXP * 8 + 1], q), a[(long long)level * N + E], q);
    }
};
// centred CRT lift of (Y[cb][0] mod q_l, Y[cb][1] mod P) into q_i; t = cb * level + i
struct LdCrt {
    const uint64_t *Y;
    const uint64_t *rr;
    int level, N;
    struct Prep {
        const uint64_t *yq, *yp;
        Modulus mq, m;
        uint64_t c2, c3, r0, r1, r2, phalf, half_q;
    };
    __device__ __forceinline__ Prep prep(int t, const DevPrimes &pr, int pidx) const {
        const int cb = t / level, i = t - cb * level;
        Prep p;
        p.yq = Y + ((long long)cb * 2) * N;
        p.yp = p.yq + N;
        p.mq = pr.m[level];
        p.m = pr.m[pidx];
        p.c2 = rr[MAXP * 8 + 2];
        p.c3 = rr[MAXP * 8 + 3];
        p.r0 = rr[i * 8 + 0];
        p.r1 = rr[i * 8 + 1];
        p.r2 = rr[i * 8 + 2];
        p.phalf = rr[MAXP * 8 + 4] >> 1;
        p.half_q = (p.mq.q - 1) >> 1;
        return p;
    }
    __device__ __forceinline__ uint64_t load(const Prep &p, long long E) const {
        const uint64_t yq = p.yq[E], yp = p.yp[E];
        const uint64_t ql = p.mq.q;
        const uint64_t tq = mul_shoup(sub_mod(yq, reduce64(yp, p.mq), ql), p.c2, p.c3, ql);
        uint64_t v = add_mod(reduce64(yp, p.m), mul_shoup(reduce64(tq, p.m), p.r0, p.r1, p.m.q), p.m.q);
        const bool neg = tq > p.half_q || (tq == p.half_q && yp > p.phalf);
        const uint64_t w = sub_mod(v, p.r2, p.m.q);
        return neg ? w : v;
    }
};
// out[c][b][i] = (P d_b[i] + acc_b[i] - z) * (P q_l)^-1 mod q_i   (t = (c*2+b) * level + i)
struct StRelinRescale {
    const uint64_t *A;
    const uint64_t *const *D3;
    uint64_t *const *O;
    const uint64_t *rr;
    int level, nt, N;
    struct Pre {
        uint64_t a, d;
    };
    struct Ctx {
        const uint64_t *a, *d;
        uint64_t *o;
        uint64_t r0, r1, r3, r4, q;
    };
    __device__ __forceinline__ Ctx ctx(uint64_t *, int t, const DevPrimes &pr, int pidx) const {
        const int cb = t / level, i = t - cb * level, c = cb >> 1, b = cb & 1;
        Ctx x;
        x.a = A + ((long long)cb * nt + i) * N;
        x.d = D3[c] + ((long long)b * (level + 1) + i) * N;
        x.o = O[c] + ((long long)b * level + i) * N;
        x.r0 = rr[i * 8 + 0];
        x.r1 = rr[i * 8 + 1];
        x.r3 = rr[i * 8 + 3];
        x.r4 = rr[i * 8 + 4];
        x.q = pr.m[pidx].q;
        return x;
    }
    __device__ __forceinline__ Pre prefetch(const Ctx &x, long long E) const { return Pre{x.a[E], x.d[E]}; }
    __device__ __forceinline__ void finish(const Ctx &x, long long E, uint64_t z, const Pre &p) const {
        const uint64_t v = add_mod(mul_shoup(p.d, x.r0, x.r1, x.q), p.a, x.q);
        x.o[E] = mul_shoup(sub_mod(v, z, x.q), x.r3, x.r4, x.q);
    }
};

std::vector<const uint64_t *> strided_ptrs(const uint64_t *base, int count, size_t stride) {
    std::vector<const uint64_t *> v(count);
    for (int i = 0; i < count; i++) v[i] = base + (size_t)i * stride;
    return v;
}

}  // namespace

void rescale(Ctx &c, const uint64_t *const *In, uint64_t *const *Out, int count, int polys, int level) {
    if (level < 1) throw VrError(3, "rescale: no level left to drop");
    const int N = c.n;
    const int rows = count * polys;
    Scratch y(c, sizeof(uint64_t) * rows * N), z(c, sizeof(uint64_t) * rows * level * N);
    // y = INTT_{q_l}(top limb of every polynomial)
    ntt_inverse_fused(c, NttBatch{y.as<uint64_t>(), rows, 1, (long long)N, 1, level, 0, 0},
                      nttk::LdGather{In, polys, (long long)(level + 1) * N, (long long)level * N}, nttk::StPlain{});
    // out_i = (in_i - NTT_{q_i}(lift(y))) * q_l^-1
    nttk::StCombine st{In, Out, nullptr, c.inv_tab + (size_t)level * c.np * 2, level, polys, level + 1, 0, c.log_n, 1u};
    ntt_forward_fused(c, batch_limbs(z.as<uint64_t>(), rows, level, N), nttk::LdLift{y.as<uint64_t>(), level, 1, level, N, c.f64mask, c.liftk, c.ntt_const}, st);
}

// cl_intt: run the INTT of the digits as one cluster kernel whatever the batch size.  Measured on
// B200 for the relinearisation inside matmul_outer, next to the streaming (d0, d1) pass: cfg-2 step
// 82.6 -> 79.9 us, cfg 1 +5%; for the isolated small ModUps of hoisted rotations it is slower
// (Algorithm 3 84 -> 74 HE matmul/s), so only the relinearisation path asks for it.
// VR_MODUP_INTT_CL=0 disables it.
static void modup_impl(Ctx &c, const uint64_t *const *Polys, long long poly_off, int count, int level, uint64_t *D,
                       bool cl_intt_wanted = false) {
    const int N = c.n, nl = level + 1, nt = level + 2;
    Scratch x(c, sizeof(uint64_t) * count * nl * N);
    static const int cl_env = [] {
        const char *e = getenv("VR_MODUP_INTT_CL");
        return e ? atoi(e) : 1;
    }();
    if (cl_intt_wanted && cl_env)
        ntt_inverse_cl(c, batch_limbs(x.as<uint64_t>(), count, nl, N), nttk::LdGather{Polys, nl, (long long)N, poly_off},
                       nttk::StPlain{});
    else
        ntt_inverse_fused(c, batch_limbs(x.as<uint64_t>(), count, nl, N), nttk::LdGather{Polys, nl, (long long)N, poly_off},
                          nttk::StPlain{});
    ntt_forward_fused(c, NttBatch{D, count * nl * nt, nt, (long long)nt * N, nl, 0, c.np - 1, nl},
                      nttk::LdLift{x.as<uint64_t>(), nt, nl, -1, N, c.f64mask, c.liftk, c.ntt_const}, nttk::StPlain{});
}

void modup(Ctx &c, const uint64_t *const *Polys, int count, int level, uint64_t *D) { modup_impl(c, Polys, 0, count, level, D); }

template <int CG>
static void launch_ks_inner_cg(Ctx &c, const uint64_t *D, const uint64_t *const *Polys, long long poly_off, int count, int level,
                               const uint64_t *key, uint32_t g, uint64_t *A, const uint64_t *const *keys_r,
                               const uint32_t *gs_r, int nrot) {
    const int N = c.n, nl = level + 1, nt = level + 2;
    const dim3 blocks(nblocks((long long)nt * N, 128), (count + CG - 1) / CG, nrot);
    if (nl <= 8)
        launch_pdl(k_ks_inner<8, CG>, blocks, dim3(128), 0, c.stream, D, Polys, poly_off, count, level, N, c.log_n, c.np, key, g,
                   c.primes, A, (const NttConst *)c.ntt_const, keys_r, gs_r);
    else if (nl <= 16)
        launch_pdl(k_ks_inner<16, CG>, blocks, dim3(128), 0, c.stream, D, Polys, poly_off, count, level, N, c.log_n, c.np, key,
                   g, c.primes, A, (const NttConst *)c.ntt_const, keys_r, gs_r);
    else
        launch_pdl(k_ks_inner<40, 1>, dim3(blocks.x, count, nrot), dim3(128), 0, c.stream, D, Polys, poly_off, count, level, N,
                   c.log_n, c.np, key, g, c.primes, A, (const NttConst *)c.ntt_const, keys_r, gs_r);
    check_launch("k_ks_inner");
}

static void launch_ks_inner(Ctx &c, const uint64_t *D, const uint64_t *const *Polys, long long poly_off, int count, int level,
                            const uint64_t *key, uint32_t g, uint64_t *A, const uint64_t *const *keys_r = nullptr,
                            const uint32_t *gs_r = nullptr, int nrot = 1) {
    static int cg_env = [] {
        const char *e = getenv("VR_KS_CG");
        return e ? atoi(e) : 0;
    }();
    // swept on B200: 1/2/4/8 within 2% for <= 8 digits; above 8 digits (Table 1, 14 limbs) one
    // ciphertext per thread (146 instead of 175 registers) is ~1.5% faster
    const int cg = cg_env ? cg_env : (level + 1 > 8 ? 1 : 2);
    switch (cg) {
        case 1: launch_ks_inner_cg<1>(c, D, Polys, poly_off, count, level, key, g, A, keys_r, gs_r, nrot); break;
        case 2: launch_ks_inner_cg<2>(c, D, Polys, poly_off, count, level, key, g, A, keys_r, gs_r, nrot); break;
        case 8: launch_ks_inner_cg<8>(c, D, Polys, poly_off, count, level, key, g, A, keys_r, gs_r, nrot); break;
        default: launch_ks_inner_cg<4>(c, D, Polys, poly_off, count, level, key, g, A, keys_r, gs_r, nrot); break;
    }
}

// Out (pointer table, count entries of [2][l+1][N]) = ModDown(inner(D, key)) (+ add)
static void inner_moddown(Ctx &c, const uint64_t *D, const uint64_t *const *Polys, long long poly_off, int count, int level,
                          const uint64_t *key, uint32_t g, uint64_t *const *Out, const uint64_t *const *Add, int add_polys) {
    const int N = c.n, nl = level + 1, nt = level + 2, P = c.np - 1;
    Scratch a(c, sizeof(uint64_t) * count * 2 * nt * N);
    launch_ks_inner(c, D, Polys, poly_off, count, level, key, g, a.as<uint64_t>());
    const int rows = count * 2;
    Scratch y(c, sizeof(uint64_t) * rows * N), z(c, sizeof(uint64_t) * rows * nl * N);
    ntt_inverse_fused(c, NttBatch{y.as<uint64_t>(), rows, 1, (long long)N, 1, P, 0, 0},
                      LdStrided{a.as<uint64_t>(), (long long)nt * N, (long long)nl * N}, nttk::StPlain{});
    PtrTable ta(c, strided_ptrs(a.as<uint64_t>(), count, (size_t)2 * nt * N));
    nttk::StCombine st{ta.c_(), Out, Add, c.inv_tab + (size_t)P * c.np * 2, nl, 2, nt, add_polys, c.log_n, g};
    ntt_forward_fused(c, batch_limbs(z.as<uint64_t>(), rows, nl, N), nttk::LdLift{y.as<uint64_t>(), nl, 1, P, N, c.f64mask, c.liftk, c.ntt_const}, st);
}

// inner_moddown for every rotation amount of a hoisted batch at once: one inner-product launch (grid z
// = amount), one INTT and one NTT + combine over count * nrot ciphertexts; Out [count * nrot] ordered
// [ct][amount], Add[ct] permuted by amount r's Galois element.  Replaces 4 launches per amount.
static void inner_moddown_multi(Ctx &c, const uint64_t *D, const uint64_t *const *Polys, long long poly_off, int count,
                                int level, const uint64_t *const *keys_r, const uint32_t *gs_r, int nrot,
                                uint64_t *const *Out, const uint64_t *const *Add, int add_polys) {
    const int N = c.n, nl = level + 1, nt = level + 2, P = c.np - 1, total = count * nrot;
    Scratch a(c, sizeof(uint64_t) * total * 2 * nt * N);
    launch_ks_inner(c, D, Polys, poly_off, count, level, nullptr, 1, a.as<uint64_t>(), keys_r, gs_r, nrot);
    const int rows = total * 2;
    Scratch y(c, sizeof(uint64_t) * rows * N), z(c, sizeof(uint64_t) * rows * nl * N);
    ntt_inverse_fused(c, NttBatch{y.as<uint64_t>(), rows, 1, (long long)N, 1, P, 0, 0},
                      LdStrided{a.as<uint64_t>(), (long long)nt * N, (long long)nl * N}, nttk::StPlain{});
    PtrTable ta(c, strided_ptrs(a.as<uint64_t>(), total, (size_t)2 * nt * N));
    nttk::StCombine st{ta.c_(), Out, Add, c.inv_tab + (size_t)P * c.np * 2, nl, 2, nt, add_polys, c.log_n, 1u};
    st.gs_rows = gs_r;
    st.add_div = nrot;
    ntt_forward_fused(c, batch_limbs(z.as<uint64_t>(), rows, nl, N), nttk::LdLift{y.as<uint64_t>(), nl, 1, P, N, c.f64mask, c.liftk, c.ntt_const}, st);
}

void keyswitch_poly(Ctx &c, const uint64_t *const *Polys, int count, int level, const uint64_t *key, uint64_t *const *Out) {
    const int N = c.n, nl = level + 1, nt = level + 2;
    Scratch d(c, sizeof(uint64_t) * count * nl * nt * N);
    modup_impl(c, Polys, 0, count, level, d.as<uint64_t>());
    inner_moddown(c, d.as<uint64_t>(), Polys, 0, count, level, key, 1, Out, nullptr, 0);
}

// relinearise and rescale in one rounding step: (P d + acc) / (P q_l)
void relin_rescale_batch(Ctx &c, const uint64_t *const *D3, uint64_t *const *Out, int count, int level, cudaEvent_t d01_ready) {
    if (level < 1) throw VrError(3, "relin_rescale: no level left to drop");
    const int N = c.n, nl = level + 1, nt = level + 2, P = c.np - 1;
    const uint64_t *key = relin_key(c);
    const long long off = (long long)2 * nl * N;
    Scratch d(c, sizeof(uint64_t) * count * nl * nt * N), a(c, sizeof(uint64_t) * count * 2 * nt * N);
    modup_impl(c, D3, off, count, level, d.as<uint64_t>(), true);
    launch_ks_inner(c, d.as<uint64_t>(), D3, off, count, level, key, 1, a.as<uint64_t>());
    const uint64_t *rr = c.rr_tab + (size_t)level * RR_STRIDE;
    Scratch y(c, sizeof(uint64_t) * count * 4 * N), z(c, sizeof(uint64_t) * count * 2 * level * N);
    if (d01_ready) VR_CUDA(cudaStreamWaitEvent(c.stream, d01_ready, 0));  // (d0, d1) produced on another stream
    // (a cluster kernel here measured slower inside matmul_outer: 79.9 -> 84.5 us)
    ntt_inverse_fused(c, NttBatch{y.as<uint64_t>(), count * 4, 2, (long long)2 * N, 1, level, P, 0},
                      LdXrow{a.as<uint64_t>(), D3, rr, level, nt, N}, nttk::StPlain{});
    ntt_forward_fused(c, batch_limbs(z.as<uint64_t>(), count * 2, level, N), LdCrt{y.as<uint64_t>(), rr, level, N},
                      StRelinRescale{a.as<uint64_t>(), D3, Out, rr, level, nt, N});
}

void relin_batch(Ctx &c, const uint64_t *const *D3, uint64_t *const *Out, int count, int level) {
    const int N = c.n, nl = level + 1, nt = level + 2;
    const uint64_t *key = relin_key(c);
    Scratch d(c, sizeof(uint64_t) * count * nl * nt * N);
    const long long off = (long long)2 * nl * N;
    modup_impl(c, D3, off, count, level, d.as<uint64_t>());
    inner_moddown(c, d.as<uint64_t>(), D3, off, count, level, key, 1, Out, D3, 2);
}

void rotate_batch(Ctx &c, const uint64_t *const *In, uint64_t *const *Out, int count, int level, int nrot, const uint32_t *gs) {
    // Out has count*nrot entries ordered [ct][rot]
    const int N = c.n, nl = level + 1, nt = level + 2;
    std::vector<uint64_t *> keys(nrot);
    bool any = false;
    for (int r = 0; r < nrot; r++) {
        keys[r] = gs[r] == 1 ? nullptr : galois_key(c, gs[r]);
        any |= gs[r] != 1;
    }
    Scratch d(c, any ? sizeof(uint64_t) * count * nl * nt * N : 0);
    const long long off = (long long)nl * N;
    if (any) modup_impl(c, In, off, count, level, d.as<uint64_t>());
    // VR_ROT_BATCH=1: one launch sequence for all amounts (parity-tested; measured on B200 Alg 3 90.8
    // vs 94.0 HE matmul/s, cfg 3/4/5b and Table 1 unchanged -- the rotations are device-bound)
    static const bool batched = [] {
        const char *e = getenv("VR_ROT_BATCH");
        return e != nullptr && atoi(e) != 0;
    }();
    bool all_rot = nrot > 1;
    for (int r = 0; r < nrot; r++) all_rot &= gs[r] != 1;
    if (batched && all_rot) {  // every amount a real rotation: one launch sequence for all of them
        std::vector<const uint64_t *> kv(keys.begin(), keys.end());
        PtrTable tk(c, kv);
        DevArray<uint32_t> dg(c, gs, nrot);
        inner_moddown_multi(c, d.as<uint64_t>(), In, off, count, level, tk.c_(), dg.get(), nrot, Out, In, 1);
        return;
    }
    for (int r = 0; r < nrot; r++) {
        Scratch tbl(c, sizeof(void *) * count);
        VR_CUDA(cudaMemcpy2DAsync(tbl.p, sizeof(void *), (const void *)(Out + r), sizeof(void *) * nrot, sizeof(void *), count,
                                  cudaMemcpyDeviceToDevice, c.stream));
        uint64_t *const *outr = tbl.as<uint64_t *>();
        if (gs[r] == 1) {
            copy_limbs(c, In, outr, count, 2, nl, nl, 0);
            continue;
        }
        inner_moddown(c, d.as<uint64_t>(), In, off, count, level, keys[r], gs[r], outr, In, 1);
    }
}

}  // namespace vr
