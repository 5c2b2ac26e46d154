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

// X[c][i][k] = P[c][poly_off + i*N + k]
__global__ void k_gather(const uint64_t *const *P, long long poly_off, int count, int nl, int N, uint64_t *X) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long per = (long long)nl * N;
    if (e >= count * per) return;
    const long long c = e / per, r = e - c * per;
    X[e] = P[c][poly_off + r];
}

// D[c][j][t][k]: t == j -> original NTT limb; else lift(X[c][j][k], q_j -> q_t) (coeff domain)
__global__ void k_modup_lift(const uint64_t *X, const uint64_t *const *P, long long poly_off, int count, int level, int N,
                             int pspecial, DevPrimes pr, uint64_t *D) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int nl = level + 1, nt = level + 2;
    if (e >= (long long)count * nl * nt * N) return;
    const int k = (int)(e % N);
    long long rest = e / N;
    const int t = (int)(rest % nt);
    rest /= nt;
    const int j = (int)(rest % nl);
    const long long c = rest / nl;
    uint64_t v;
    if (t == j) v = P[c][poly_off + (long long)j * N + k];
    else {
        const int pidx = t < nl ? t : pspecial;
        v = lift_centered(X[(c * nl + j) * N + k], pr.m[j].q, pr.m[pidx]);
    }
    D[e] = v;
}

// A[c][x][t][k] = sum_j D[c][j][t][src(k)] * key[j][x][pidx(t)][k]
__global__ void k_ks_inner(const uint64_t *D, int count, int level, int N, int logN, int np, const uint64_t *key, uint32_t g,
                           DevPrimes pr, uint64_t *A) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int nl = level + 1, nt = level + 2;
    if (e >= (long long)count * nt * N) return;
    const int k = (int)(e % N);
    long long rest = e / N;
    const int t = (int)(rest % nt);
    const long long c = rest / nt;
    const int pidx = t < nl ? t : np - 1;
    const Modulus m = pr.m[pidx];
    const int src = galois_src(k, g, logN);
    u128 a0{0, 0}, a1{0, 0};
    for (int j = 0; j < nl; j++) {
        const uint64_t d = D[((c * nl + j) * nt + t) * N + src];
        const uint64_t k0 = key[(((size_t)j * 2 + 0) * np + pidx) * N + k];
        const uint64_t k1 = key[(((size_t)j * 2 + 1) * np + pidx) * N + k];
        mac_to(a0, d, k0);
        mac_to(a1, d, k1);
        if ((j & 7) == 7) { a0 = u128{reduce128(a0, m), 0}; a1 = u128{reduce128(a1, m), 0}; }
    }
    A[((c * 2 + 0) * nt + t) * N + k] = reduce128(a0, m);
    A[((c * 2 + 1) * nt + t) * N + k] = reduce128(a1, m);
}

// Y[r][k] = A[r][last][k] for r in count*2 polys of nt limbs
__global__ void k_pick_limb(const uint64_t *A, int rows, int nt, int limb, int N, uint64_t *Y) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)rows * N) return;
    const long long r = e / N;
    const int k = (int)(e - r * N);
    Y[e] = A[(r * nt + limb) * N + k];
}

// Z[r][i][k] = lift(Y[r][k], from -> q_i), i < nout
__global__ void k_lift_rows(const uint64_t *Y, int rows, int nout, int N, uint64_t from, DevPrimes pr, uint64_t *Z) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)rows * nout * N) return;
    const int k = (int)(e % N);
    const long long ri = e / N;
    const int i = (int)(ri % nout);
    const long long r = ri / nout;
    Z[e] = lift_centered(Y[r * N + k], from, pr.m[i]);
}

// Out[r][i][k] = (A[r][i][k] - Z[r][i][k]) * inv_i   with A rows of nt limbs
__global__ void k_sub_mul(const uint64_t *A, int nt, const uint64_t *Z, int rows, int nout, int N, const uint64_t *inv_row,
                          DevPrimes pr, uint64_t *Out) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)rows * nout * N) return;
    const int k = (int)(e % N);
    const long long ri = e / N;
    const int i = (int)(ri % nout);
    const long long r = ri / nout;
    const uint64_t q = pr.m[i].q;
    const uint64_t a = A[(r * nt + i) * N + k];
    Out[e] = mul_shoup(sub_mod(a, Z[e], q), inv_row[2 * i], inv_row[2 * i + 1], q);
}

// rescale inputs come through a pointer table: Y[c*polys+p][k] = In[c][(p*(l+1) + l)*N + k]
__global__ void k_pick_top(const uint64_t *const *In, int count, int polys, int level, int N, uint64_t *Y) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)count * polys * N) return;
    const long long r = e / N;
    const int k = (int)(e - r * N);
    const long long c = r / polys;
    const int p = (int)(r - c * polys);
    Y[e] = In[c][((size_t)p * (level + 1) + level) * N + k];
}

__global__ void k_rescale_combine(const uint64_t *const *In, const uint64_t *Z, int count, int polys, int level, int N,
                                  const uint64_t *inv_row, DevPrimes pr, uint64_t *const *Out) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)count * polys * level * N) return;
    const int k = (int)(e % N);
    long long rest = e / N;
    const int i = (int)(rest % level);
    rest /= level;
    const int p = (int)(rest % polys);
    const long long c = rest / polys;
    const uint64_t q = pr.m[i].q;
    const uint64_t a = In[c][((size_t)p * (level + 1) + i) * N + k];
    Out[c][((size_t)p * level + i) * N + k] = mul_shoup(sub_mod(a, Z[e], q), inv_row[2 * i], inv_row[2 * i + 1], q);
}

// Out[c][0] = perm_g(In[c][0]) + KS[c][0];  Out[c][1] = KS[c][1]
__global__ void k_rot_finish(const uint64_t *const *In, const uint64_t *KS, int count, int nl, int N, int logN, uint32_t g,
                             DevPrimes pr, uint64_t *const *Out) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)count * 2 * nl * N) return;
    const int k = (int)(e % N);
    long long rest = e / N;
    const int i = (int)(rest % nl);
    rest /= nl;
    const int p = (int)(rest % 2);
    const long long c = rest / 2;
    uint64_t v = KS[e];
    if (p == 0) v = add_mod(v, In[c][(size_t)i * N + galois_src(k, g, logN)], pr.m[i].q);
    Out[c][((size_t)p * nl + i) * N + k] = v;
}

}  // namespace

void rescale(Ctx &c, const uint64_t *const *In, uint64_t *const *Out, int count, int polys, int level) {
    if (level < 1) throw VrError(3, "rescale: no level left to drop");
    const int N = c.n;
    const long long rows = (long long)count * polys;
    Scratch y(c, sizeof(uint64_t) * rows * N), z(c, sizeof(uint64_t) * rows * level * N);
    k_pick_top<<<nblocks(rows * N, TB), TB, 0, c.stream>>>(In, count, polys, level, N, y.as<uint64_t>());
    check_launch("k_pick_top");
    ntt_inverse(c, NttBatch{y.as<uint64_t>(), (int)rows, 1, (long long)N, 1, level, 0, 0});
    k_lift_rows<<<nblocks(rows * level * N, TB), TB, 0, c.stream>>>(y.as<uint64_t>(), (int)rows, level, N, c.q[level],
                                                                     c.primes, z.as<uint64_t>());
    check_launch("k_lift_rows");
    ntt_forward(c, batch_limbs(z.as<uint64_t>(), (int)rows, level, N));
    const uint64_t *inv_row = c.inv_tab + (size_t)level * c.np * 2;
    k_rescale_combine<<<nblocks(rows * level * N, TB), TB, 0, c.stream>>>(In, z.as<uint64_t>(), count, polys, level, N,
                                                                           inv_row, c.primes, Out);
    check_launch("k_rescale_combine");
}

static void modup_impl(Ctx &c, const uint64_t *const *Polys, long long poly_off, int count, int level, uint64_t *D) {
    const int N = c.n, nl = level + 1, nt = level + 2;
    Scratch x(c, sizeof(uint64_t) * count * nl * N);
    k_gather<<<nblocks((long long)count * nl * N, TB), TB, 0, c.stream>>>(Polys, poly_off, count, nl, N, x.as<uint64_t>());
    check_launch("k_gather");
    ntt_inverse(c, batch_limbs(x.as<uint64_t>(), count, nl, N));
    k_modup_lift<<<nblocks((long long)count * nl * nt * N, TB), TB, 0, c.stream>>>(x.as<uint64_t>(), Polys, poly_off, count,
                                                                                    level, N, c.np - 1, c.primes, D);
    check_launch("k_modup_lift");
    ntt_forward(c, NttBatch{D, count * nl * nt, nt, (long long)nt * N, nl, 0, c.np - 1, nl});
}

void modup(Ctx &c, const uint64_t *const *Polys, int count, int level, uint64_t *D) { modup_impl(c, Polys, 0, count, level, D); }

void ks_inner_moddown(Ctx &c, const uint64_t *D, int count, int level, const uint64_t *key, uint32_t g, uint64_t *Out) {
    const int N = c.n, nl = level + 1, nt = level + 2;
    Scratch a(c, sizeof(uint64_t) * count * 2 * nt * N);
    k_ks_inner<<<nblocks((long long)count * nt * N, TB), TB, 0, c.stream>>>(D, count, level, N, c.log_n, c.np, key, g,
                                                                            c.primes, a.as<uint64_t>());
    check_launch("k_ks_inner");
    const int rows = count * 2;
    Scratch y(c, sizeof(uint64_t) * rows * N), z(c, sizeof(uint64_t) * rows * nl * N);
    k_pick_limb<<<nblocks((long long)rows * N, TB), TB, 0, c.stream>>>(a.as<uint64_t>(), rows, nt, nl, N, y.as<uint64_t>());
    check_launch("k_pick_limb");
    const int P = c.np - 1;
    ntt_inverse(c, NttBatch{y.as<uint64_t>(), rows, 1, (long long)N, 1, P, 0, 0});
    k_lift_rows<<<nblocks((long long)rows * nl * N, TB), TB, 0, c.stream>>>(y.as<uint64_t>(), rows, nl, N, c.q[P], c.primes,
                                                                            z.as<uint64_t>());
    check_launch("k_lift_rows");
    ntt_forward(c, batch_limbs(z.as<uint64_t>(), rows, nl, N));
    const uint64_t *inv_row = c.inv_tab + (size_t)P * c.np * 2;
    k_sub_mul<<<nblocks((long long)rows * nl * N, TB), TB, 0, c.stream>>>(a.as<uint64_t>(), nt, z.as<uint64_t>(), rows, nl, N,
                                                                          inv_row, c.primes, Out);
    check_launch("k_sub_mul");
}

void relin_batch(Ctx &c, const uint64_t *const *D3, uint64_t *const *Out, int count, int level) {
    const int N = c.n, nl = level + 1, nt = level + 2;
    const uint64_t *key = relin_key(c);
    Scratch d(c, sizeof(uint64_t) * count * nl * nt * N), ks(c, sizeof(uint64_t) * count * 2 * nl * N);
    modup_impl(c, D3, (long long)2 * nl * N, count, level, d.as<uint64_t>());
    ks_inner_moddown(c, d.as<uint64_t>(), count, level, key, 1, ks.as<uint64_t>());
    std::vector<const uint64_t *> kp(count);
    for (int i = 0; i < count; i++) kp[i] = ks.as<uint64_t>() + (size_t)i * 2 * nl * N;
    PtrTable kt(c, kp);
    binop(c, D3, kt.c_(), Out, count, 2, nl, 0);
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
    Scratch d(c, any ? sizeof(uint64_t) * count * nl * nt * N : 0), ks(c, sizeof(uint64_t) * count * 2 * nl * N);
    if (any) modup_impl(c, In, (long long)nl * N, count, level, d.as<uint64_t>());
    // device copy of Out table, needed per rotation with stride nrot
    std::vector<uint64_t *> hostOut(count);
    for (int r = 0; r < nrot; r++) {
        // gather the output pointers for this rotation amount
        Scratch tbl(c, sizeof(void *) * count);
        VR_CUDA(cudaMemcpy2DAsync(tbl.p, sizeof(void *), (const void *)(Out + r), sizeof(void *) * nrot, sizeof(void *), count,
                                  cudaMemcpyDeviceToDevice, c.stream));
        uint64_t *const *outr = tbl.as<uint64_t *>();
        if (gs[r] == 1) {
            copy_limbs(c, In, outr, count, 2, nl, nl, 0);
            continue;
        }
        ks_inner_moddown(c, d.as<uint64_t>(), count, level, keys[r], gs[r], ks.as<uint64_t>());
        k_rot_finish<<<nblocks((long long)count * 2 * nl * N, TB), TB, 0, c.stream>>>(In, ks.as<uint64_t>(), count, nl, N,
                                                                                       c.log_n, gs[r], c.primes, outr);
        check_launch("k_rot_finish");
    }
}

}  // namespace vr
