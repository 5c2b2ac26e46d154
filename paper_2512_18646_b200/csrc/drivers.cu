// drivers.cu -- batched column-ciphertext drivers.
//
//   matmul_outer   multicipher.py:88-103   sum_k tensor(L_k, R_k) in one pass,
//                                           then ONE relinearisation + ONE rescale
//   conv_columns   multicipher.py:123-162  hoisted rotations shared by every
//                                           filter/output column, one MAC kernel
//                                           for all (filter, column, channel, tap)
//   poly_activation pipeline.py:180-197    the same op sequence for a whole batch
//
// Each driver restates the op order of the matching oracle/ckks_oracle.c
// function, so residues are bit-identical to the CPU oracle.
#include <algorithm>
#include <map>

#include "encode.cuh"

namespace vr {

namespace {

constexpr int TB = 256;

std::vector<const uint64_t *> strided(const uint64_t *base, int count, size_t stride) {
    std::vector<const uint64_t *> v(count);
    for (int i = 0; i < count; i++) v[i] = base + (size_t)i * stride;
    return v;
}

// Conv MAC: Yp[f][o] = mask * (sum_{c,q,p} w[f][c][p][q] * T[c][cols[o]+q][p] + bias[f])
template <int FG>
__global__ void __launch_bounds__(128) k_conv_mac(const uint64_t *const *T, const int *cols, int nout, int C, int W, int k,
                                                  int F, const uint64_t *wq, const uint64_t *bq, const uint64_t *mask, int nl,
                                                  int N, DevPrimes pr, uint64_t *Yp) {
    pdl_wait();
    pdl_trigger();
    const int kk = blockIdx.z * blockDim.x + threadIdx.x;
    if (kk >= N) return;
    const int poly = blockIdx.y / nl, i = blockIdx.y - poly * nl;
    const int nfg = F / FG;
    const int o = blockIdx.x / nfg, f0 = (blockIdx.x - o * nfg) * FG;
    const Modulus m = pr.m[i];
    u128 acc[FG];
#pragma unroll
    for (int f = 0; f < FG; f++) acc[f] = u128{0, 0};
    int cnt = 0;
    const size_t off = ((size_t)poly * nl + i) * N + kk;
    const int kk2 = k * k;
    for (int c = 0; c < C; c++)
        for (int q = 0; q < k; q++) {
            const int j = cols[o] + q;
            for (int p = 0; p < k; p++) {
                const uint64_t *src = T[((size_t)c * W + j) * k + p];
                if (!src) continue;
                const uint64_t v = src[off];
                const uint64_t *wr = wq + (((size_t)i * F + f0) * C + c) * kk2 + p * k + q;
#pragma unroll
                for (int f = 0; f < FG; f++) mac_to(acc[f], v, __ldg(wr + (size_t)f * C * kk2));
                if (++cnt == 16) {
                    cnt = 0;
#pragma unroll
                    for (int f = 0; f < FG; f++) acc[f] = u128{reduce128(acc[f], m), 0};
                }
            }
        }
    const uint64_t mk = mask[(size_t)i * N + kk];
#pragma unroll
    for (int f = 0; f < FG; f++) {
        uint64_t r = reduce128(acc[f], m);
        if (poly == 0) r = add_mod(r, bq[(size_t)i * F + f0 + f], m.q);
        r = mul_mod(r, mk, m);
        Yp[((size_t)(f0 + f) * nout + o) * 2 * nl * N + off] = r;
    }
}

__device__ __forceinline__ ulonglong2 ld2(const uint64_t *p) { return *reinterpret_cast<const ulonglong2 *>(p); }
__device__ __forceinline__ void st2(uint64_t *p, uint64_t a, uint64_t b) {
    *reinterpret_cast<ulonglong2 *>(p) = make_ulonglong2(a, b);
}

// Small-weight conv MAC.  Quantised weights satisfy |w| < B = 2^bb, so w' = w + B
// is a u32.  Splitting each residue v = vh * 2^32 + vl, every product w' * v is
// accumulated as two 32x32+64 multiply-adds (IMAD.WIDE.U32) into 64-bit partial
// sums, which the host guarantees cannot overflow for this tap count; the bias
// B * sum(v) is shared by all filters and removed once at the end.  A thread owns
// two adjacent coefficients (16-byte loads) and FG filters; pointers and weights
// of the CTA's output column are staged in shared memory (weights read as 16 B).
template <int FG>
__global__ void __launch_bounds__(128) k_conv_mac_small(const uint64_t *const *T, const int *cols, int nout, int C, int W,
                                                        int k, int F, const uint32_t *wb, uint64_t bb_pow, const uint64_t *bq,
                                                        const uint64_t *mask, int nl, int N, DevPrimes pr, uint64_t *Yp) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(16) uint64_t smc[];
    const int taps = C * k * k, tpad = (taps + 3) & ~3;  // the tap list padded to a multiple of four
    const uint64_t **sptr = (const uint64_t **)smc;
    uint32_t *sw = (uint32_t *)(smc + tpad);  // [tpad][FG], 16-byte aligned rows for FG % 4 == 0
    const int nfg = F / FG;
    const int o = blockIdx.x / nfg, f0 = (blockIdx.x - o * nfg) * FG;
    for (int t = threadIdx.x; t < tpad; t += blockDim.x) {
        if (t >= taps) {
            sptr[t] = nullptr;
            for (int f = 0; f < FG; f++) sw[t * FG + f] = 0;
            continue;
        }
        const int c = t / (k * k), r = t - c * k * k, q = r / k, p = r - q * k;  // tap order (c, q, p)
        sptr[t] = T[((size_t)c * W + cols[o] + q) * k + p];
        for (int f = 0; f < FG; f++) sw[t * FG + f] = wb[((size_t)(f0 + f) * C + c) * k * k + p * k + q];
    }
    __syncthreads();
    const int kk = (blockIdx.z * blockDim.x + threadIdx.x) * 2;
    if (kk >= N) return;
    const int poly = blockIdx.y / nl, i = blockIdx.y - poly * nl;
    const Modulus m = pr.m[i];
    const size_t off = ((size_t)poly * nl + i) * N + kk;
    uint64_t alo[2][FG], ahi[2][FG];
#pragma unroll
    for (int f = 0; f < FG; f++) alo[0][f] = ahi[0][f] = alo[1][f] = ahi[1][f] = 0;
    // Four taps per iteration: their 16-byte loads are issued together, then 4 x 4 FG multiply-adds in
    // the fused form (mad.wide.u32, 64-bit accumulator in place).  The tap list is padded to a multiple
    // of four with null pointers (value 0: nothing is added to the accumulators or to sum(v)), so the
    // loop has no guards; a null tap of the model (all-zero weights) reads as 0 the same way.
    u128 sv[2] = {u128{0, 0}, u128{0, 0}};  // sum of the tap values (bias removal)
    const int taps4 = (taps + 3) & ~3;
    for (int t0 = 0; t0 < taps4; t0 += 4) {
        ulonglong2 vv[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const uint64_t *src = sptr[t0 + u];  // CTA-uniform
            vv[u] = src ? ld2(src + off) : make_ulonglong2(0, 0);
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            uint32_t wv[FG];
#pragma unroll
            for (int f = 0; f < FG; f += (FG >= 4 ? 4 : 1)) {
                if (FG >= 4) {
                    const uint4 w4 = *reinterpret_cast<const uint4 *>(sw + (t0 + u) * FG + f);
                    wv[f] = w4.x; wv[f + 1] = w4.y; wv[f + 2] = w4.z; wv[f + 3] = w4.w;
                } else {
                    wv[f] = sw[(t0 + u) * FG + f];
                }
            }
            const uint64_t v2[2] = {vv[u].x, vv[u].y};
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const uint32_t vl = (uint32_t)v2[e], vh = (uint32_t)(v2[e] >> 32);
                asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, 0;" : "+l"(sv[e].lo), "+l"(sv[e].hi) : "l"(v2[e]));
#pragma unroll
                for (int f = 0; f < FG; f++) {
                    asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(alo[e][f]) : "r"(vl), "r"(wv[f]));
                    asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(ahi[e][f]) : "r"(vh), "r"(wv[f]));
                }
            }
        }
    }
    const uint64_t bq_pow = reduce64(bb_pow, m);
    const ulonglong2 mk2 = *reinterpret_cast<const ulonglong2 *>(mask + (size_t)i * N + kk);
    const uint64_t mk[2] = {mk2.x, mk2.y};
    uint64_t outv[FG][2];
#pragma unroll
    for (int e = 0; e < 2; e++) {
        const uint64_t bias_sum = mul_mod(reduce128(sv[e], m), bq_pow, m);  // B * sum(v) mod q
#pragma unroll
        for (int f = 0; f < FG; f++) {
            u128 acc{alo[e][f], 0};
            add_to(acc, u128{ahi[e][f] << 32, ahi[e][f] >> 32});
            uint64_t r = sub_mod(reduce128(acc, m), bias_sum, m.q);
            if (poly == 0) r = add_mod(r, bq[(size_t)i * F + f0 + f], m.q);
            outv[f][e] = mul_mod(r, mk[e], m);
        }
    }
#pragma unroll
    for (int f = 0; f < FG; f++)
        *reinterpret_cast<ulonglong2 *>(Yp + ((size_t)(f0 + f) * nout + o) * 2 * nl * N + off) = make_ulonglong2(outv[f][0], outv[f][1]);
}

// Plaintext mat-vec: Yp[u] = sum_j PT[u*nx + j] (.) X[j] (both polys), 128-bit accumulation.
// HBM-bound on the plaintext stream (cfg 3 dense 845->64: 2.2 GB per pass).  A thread owns two
// adjacent coefficients (16-byte loads) of one limb for UG outputs; the CTA stages the pointers of
// a chunk of JC inputs in shared memory (no dependent pointer load in the loop) and the j loop is
// unrolled by two so the next input's loads are in flight during the current MACs.
constexpr int PMV_JC = 128;
template <int UG, int JU>
__global__ void __launch_bounds__(128) k_pt_matvec(const uint64_t *const *X, int nx, const uint64_t *const *PT, int ny, int nl,
                                                   int N, DevPrimes pr, uint64_t *Yp) {
    __shared__ const uint64_t *sp[PMV_JC][UG + 1];  // [j][u] plaintext pointers, [j][UG] the input
    pdl_wait();
    pdl_trigger();
    const int kk = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
    const int i = blockIdx.y;
    const int u0 = blockIdx.z * UG;
    const Modulus m = pr.m[i];
    const size_t o0 = (size_t)i * N + kk, o1 = (size_t)(nl + i) * N + kk;
    const bool live = kk < N;
    u128 acc[UG][2][2];  // [output][poly][coefficient]
#pragma unroll
    for (int u = 0; u < UG; u++)
#pragma unroll
        for (int p = 0; p < 2; p++) acc[u][p][0] = acc[u][p][1] = u128{0, 0};
    for (int jc = 0; jc < nx; jc += PMV_JC) {
        const int nj = min(PMV_JC, nx - jc);
        __syncthreads();
        for (int t = threadIdx.x; t < nj * (UG + 1); t += blockDim.x) {
            const int jj = t / (UG + 1), u = t - jj * (UG + 1);
            sp[jj][u] = u == UG ? X[jc + jj] : (u0 + u < ny ? PT[(size_t)(u0 + u) * nx + jc + jj] : nullptr);
        }
        __syncthreads();
        if (!live) continue;
#pragma unroll JU
        for (int jj = 0; jj < nj; jj++) {
            const ulonglong2 x0 = ld2(sp[jj][UG] + o0), x1 = ld2(sp[jj][UG] + o1);
            ulonglong2 pt[UG];
#pragma unroll
            for (int u = 0; u < UG; u++) pt[u] = sp[jj][u] ? ld2(sp[jj][u] + o0) : make_ulonglong2(0, 0);
#pragma unroll
            for (int u = 0; u < UG; u++) {
                mac_to(acc[u][0][0], pt[u].x, x0.x);
                mac_to(acc[u][0][1], pt[u].y, x0.y);
                mac_to(acc[u][1][0], pt[u].x, x1.x);
                mac_to(acc[u][1][1], pt[u].y, x1.y);
            }
            if (((jc + jj) & 7) == 7) {
#pragma unroll
                for (int u = 0; u < UG; u++)
#pragma unroll
                    for (int p = 0; p < 2; p++)
#pragma unroll
                        for (int e = 0; e < 2; e++) acc[u][p][e] = u128{reduce128(acc[u][p][e], m), 0};
            }
        }
    }
    if (!live) return;
#pragma unroll
    for (int u = 0; u < UG; u++) {
        if (u0 + u >= ny) break;
        uint64_t *y = Yp + (size_t)(u0 + u) * 2 * nl * N;
        st2(y + o0, reduce128(acc[u][0][0], m), reduce128(acc[u][0][1], m));
        st2(y + o1, reduce128(acc[u][1][0], m), reduce128(acc[u][1][1], m));
    }
}

}  // namespace

void mul_batch(Ctx &c, const uint64_t *const *A, const uint64_t *const *B, uint64_t *const *Out, int count, int level) {
    const int N = c.n, nl = level + 1;
    Scratch d3(c, sizeof(uint64_t) * count * 3 * nl * N);
    PtrTable td(c, strided(d3.as<uint64_t>(), count, (size_t)3 * nl * N));
    tensor(c, A, B, td.m_(), count, nl);
    relin_rescale_batch(c, td.c_(), Out, count, level);
}

void matmul_outer(Ctx &c, const uint64_t *const *L, const uint64_t *const *R, int n, int nb, int level, uint64_t *const *Out,
                  bool one_pass) {
    const int N = c.n, nl = level + 1;
    Scratch d3(c, sizeof(uint64_t) * nb * 3 * nl * N);
    PtrTable td(c, strided(d3.as<uint64_t>(), nb, (size_t)3 * nl * N));
    static const int mm_order = [] {
        const char *e = getenv("VR_MM_ORDER");
        return e ? atoi(e) : 4;
    }();
    if (nb == 1 && n >= 8 && mm_order != 5 && !one_pass) {  // 5: one (d0, d1, d2) pass, then the chain, one stream
        // overlap: d2 = sum L1 R1 (half the operand bytes) feeds the key switch, while (d0, d1)
        // accumulate on the auxiliary stream; the final combine waits for them.  VR_MM_ORDER:
        // 4 (default, measured best: 87.7 vs 94 us at cfg 2) d2 + key switch on the highest-priority
        // stream, so their CTAs are placed before the concurrent (d0, d1) pass; 0 both sums forked
        // together, chain on the caller's stream; 1/3 d2 first then fork; 2/3 chain on the
        // high-priority stream.
        static const int order = [] {
            const char *e = getenv("VR_MM_ORDER");
            return e ? atoi(e) : 4;
        }();
        StreamScope scope(c);  // restores c.stream (and joins aux/hi on an error) on every exit
        cudaStream_t main = scope.main;
        if (order == 4) {
            // d2 and its key switch on the highest-priority stream (the block scheduler places their
            // CTAs before those of the concurrent (d0, d1) pass on the auxiliary stream)
            VR_CUDA(cudaEventRecord(c.ev_fork, main));
            VR_CUDA(cudaStreamWaitEvent(c.hi, c.ev_fork, 0));
            VR_CUDA(cudaStreamWaitEvent(c.aux, c.ev_fork, 0));
            c.stream = c.hi;
            tensor_sum_mode(c, L, R, n, nb, nl, td.m_(), 1);
            c.stream = c.aux;
            tensor_sum_mode(c, L, R, n, nb, nl, td.m_(), 2);
            VR_CUDA(cudaEventRecord(c.ev_join, c.aux));
            c.stream = c.hi;
            relin_rescale_batch(c, td.c_(), Out, nb, level, c.ev_join);
            VR_CUDA(cudaEventRecord(c.ev_hi_done, c.hi));
            c.stream = main;
            VR_CUDA(cudaStreamWaitEvent(main, c.ev_hi_done, 0));
            return;
        }
        const bool d2_first = order == 1 || order == 3;
        if (d2_first) tensor_sum_mode(c, L, R, n, nb, nl, td.m_(), 1);
        VR_CUDA(cudaEventRecord(c.ev_fork, c.stream));
        VR_CUDA(cudaStreamWaitEvent(c.aux, c.ev_fork, 0));
        c.stream = c.aux;
        tensor_sum_mode(c, L, R, n, nb, nl, td.m_(), 2);
        VR_CUDA(cudaEventRecord(c.ev_join, c.aux));
        c.stream = main;
        if (!d2_first) tensor_sum_mode(c, L, R, n, nb, nl, td.m_(), 1);
        if (order >= 2) {
            // the latency-bound key-switch chain on the highest-priority stream
            VR_CUDA(cudaEventRecord(c.ev_hi, main));
            VR_CUDA(cudaStreamWaitEvent(c.hi, c.ev_hi, 0));
            c.stream = c.hi;
            relin_rescale_batch(c, td.c_(), Out, nb, level, c.ev_join);
            VR_CUDA(cudaEventRecord(c.ev_hi_done, c.hi));
            c.stream = main;
            VR_CUDA(cudaStreamWaitEvent(main, c.ev_hi_done, 0));
            return;
        }
        relin_rescale_batch(c, td.c_(), Out, nb, level, c.ev_join);
        return;
    }
    tensor_sum(c, L, R, n, nb, nl, td.m_());
    relin_rescale_batch(c, td.c_(), Out, nb, level);
}

// B independent matmul_outer products (multicipher.py:88-103 applied to B operand pairs of the same
// n and level) as one launch sequence: one tensor-sum launch over all pairs, then one relinearise +
// rescale chain over the B degree-2 sums.  Small products (config 1) are bound by kernel launches, not
// by bytes: six launches then serve B products instead of one.  Residues are those of B separate calls.
void matmul_outer_many(Ctx &c, const uint64_t *const *L, const uint64_t *const *R, int n, int B, int level, uint64_t *const *Out) {
    const int N = c.n, nl = level + 1;
    Scratch d3(c, sizeof(uint64_t) * B * 3 * nl * N);
    PtrTable td(c, strided(d3.as<uint64_t>(), B, (size_t)3 * nl * N));
    tensor_sum_many(c, L, R, n, B, nl, td.m_());
    relin_rescale_batch(c, td.c_(), Out, B, level);
}

void conv_columns(Ctx &c, const std::vector<const uint64_t *> &X, int C, int W, int k, const int64_t *w, const uint64_t *bias,
                  int F, const int *out_cols, int nout, const uint64_t *mask_pt, int level, const std::vector<uint64_t *> &Y) {
    const int N = c.n, nl = level + 1;
    const size_t ctw = (size_t)2 * nl * N;
    // 1. which rotations are needed: (ch, j, p) with p >= 1 and some nonzero tap reading it
    std::vector<std::vector<int>> need((size_t)C * W);
    for (int ch = 0; ch < C; ch++)
        for (int j = 0; j < W; j++)
            for (int p = 1; p < k; p++) {
                bool nd = false;
                for (int f = 0; f < F && !nd; f++)
                    for (int q = 0; q < k && !nd; q++) {
                        if (w[(((size_t)f * C + ch) * k + p) * k + q] == 0) continue;
                        for (int o = 0; o < nout; o++)
                            if (out_cols[o] + q == j) { nd = true; break; }
                    }
                if (nd) need[(size_t)ch * W + j].push_back(p);
            }
    // rotated copies, grouped by identical rotation set so each group is one hoisted batch
    size_t nrot_total = 0;
    for (auto &v : need) nrot_total += v.size();
    Scratch rot(c, sizeof(uint64_t) * std::max<size_t>(nrot_total, 1) * ctw);
    std::vector<const uint64_t *> table((size_t)C * W * k, nullptr);
    std::map<std::vector<int>, std::vector<int>> groups;
    for (int cj = 0; cj < C * W; cj++) {
        table[(size_t)cj * k] = X[cj];
        if (!need[cj].empty()) groups[need[cj]].push_back(cj);
    }
    size_t slot = 0;
    const size_t d_bytes_per_ct = sizeof(uint64_t) * (size_t)nl * (nl + 1) * N;
    const int chunk = (int)std::max<size_t>(1, std::min<size_t>(256, ((size_t)2 << 30) / d_bytes_per_ct));
    for (auto &kv : groups) {
        const std::vector<int> &ps = kv.first;
        const std::vector<int> &cts = kv.second;
        std::vector<uint32_t> gs(ps.size());
        for (size_t r = 0; r < ps.size(); r++) {
            const int64_t S = c.slots;
            int64_t st = ((ps[r] % S) + S) % S;
            uint64_t g = 1;
            for (int64_t t = 0; t < st; t++) g = (g * 5) % (2ull * N);
            gs[r] = (uint32_t)g;
        }
        for (size_t b0 = 0; b0 < cts.size(); b0 += chunk) {
            const int cnt = (int)std::min<size_t>(chunk, cts.size() - b0);
            std::vector<const uint64_t *> in(cnt), outs((size_t)cnt * ps.size());
            for (int t = 0; t < cnt; t++) {
                const int cj = cts[b0 + t];
                in[t] = X[cj];
                for (size_t r = 0; r < ps.size(); r++) {
                    uint64_t *dst = rot.as<uint64_t>() + (slot++) * ctw;
                    outs[(size_t)t * ps.size() + r] = dst;
                    table[(size_t)cj * k + ps[r]] = dst;
                }
            }
            PtrTable ti(c, in), to(c, outs);
            rotate_batch(c, ti.c_(), to.m_(), cnt, level, (int)ps.size(), gs.data());
        }
    }
    // 2. weights / bias reduced per limb
    std::vector<uint64_t> wq((size_t)nl * F * C * k * k), bq((size_t)nl * F);
    for (int i = 0; i < nl; i++) {
        const Modulus &m = c.primes.m[i];
        for (size_t t = 0; t < (size_t)F * C * k * k; t++) wq[(size_t)i * F * C * k * k + t] = from_i64(w[t], m);
        for (int f = 0; f < F; f++) bq[(size_t)i * F + f] = reduce64(bias[(size_t)f * nl + i], m);
    }
    DevArray<uint64_t> dwq(c, wq.data(), wq.size()), dbq(c, bq.data(), bq.size());
    DevArray<int> dcols(c, out_cols, nout);
    PtrTable tt(c, table);
    // 3. MAC + mask into pre-rescale buffer (chunked over output columns), then rescale
    // small-weight fast path: |w| < 2^bb with bb <= 30
    int64_t wmax = 0;
    for (size_t t = 0; t < (size_t)F * C * k * k; t++) wmax = std::max<int64_t>(wmax, w[t] < 0 ? -w[t] : w[t]);
    int bb = 1;
    while ((int64_t(1) << bb) <= wmax) bb++;
    const int taps_total = C * k * k;
    // 64-bit partials: 2^32 * 2^(bb+1) * taps < 2^64  (and sum(v) halves: taps < 2^31)
    const bool small = bb <= 30 && (int64_t)taps_total <= (int64_t(1) << (31 - bb)) && N >= 2;
    std::vector<uint32_t> wbias;
    int flush = 1;
    if (small) {
        wbias.resize((size_t)F * C * k * k);
        for (size_t t = 0; t < wbias.size(); t++) wbias[t] = (uint32_t)(w[t] + (int64_t(1) << bb));
        flush = taps_total;
    }
    DevArray<uint32_t> dwb(c, small ? wbias.data() : nullptr, small ? wbias.size() : 0);
    const int taps = C * k * k;
    static const int fg_max = [] {
        const char *e = getenv("VR_CONV_FG");
        return e ? atoi(e) : 8;
    }();
    const int FG = (F % 8 == 0 && fg_max >= 8) ? 8 : (F % 4 == 0 && fg_max >= 4 ? 4 : (F % 2 == 0 && fg_max >= 2 ? 2 : 1));
    const int ocols = std::max(1, std::min(nout, (int)(((size_t)2 << 30) / (ctw * 8 * F))));
    Scratch yp(c, sizeof(uint64_t) * (size_t)F * ocols * ctw);
    for (int o0 = 0; o0 < nout; o0 += ocols) {
        const int no = std::min(ocols, nout - o0);
        // grid x = (output column, filter group) fastest, z = coefficient tile: CTAs resident together
        // share one coefficient tile, so a rotated tap read by k output columns and F / FG filter
        // groups is served from L2 after its first read (measured 5.35 -> 5.19 ms per cfg-4 launch;
        // the MAC is instruction-bound: ncu 3.2 G warp instructions, 7x the IMAD.WIDE count)
        dim3 grid((unsigned)no * (F / FG), 2 * nl, nblocks(N, 128));
        const int *colp = dcols.get() + o0;
        if (small) {
            const size_t tpad = (size_t)((taps + 3) & ~3);
            const size_t sm = tpad * 8 + tpad * FG * 4 + 16;
            const uint64_t bpow = uint64_t(1) << bb;
            dim3 gs((unsigned)no * (F / FG), 2 * nl, nblocks(N / 2, 128));
            switch (FG) {
                case 8: launch_pdl(k_conv_mac_small<8>, dim3(gs), dim3(128), sm, c.stream, tt.c_(), colp, no, C, W, k, F, dwb.get(), bpow, dbq.get(), mask_pt, nl, N, c.primes, yp.as<uint64_t>()); break;
                case 4: launch_pdl(k_conv_mac_small<4>, dim3(gs), dim3(128), sm, c.stream, tt.c_(), colp, no, C, W, k, F, dwb.get(), bpow, dbq.get(), mask_pt, nl, N, c.primes, yp.as<uint64_t>()); break;
                case 2: launch_pdl(k_conv_mac_small<2>, dim3(gs), dim3(128), sm, c.stream, tt.c_(), colp, no, C, W, k, F, dwb.get(), bpow, dbq.get(), mask_pt, nl, N, c.primes, yp.as<uint64_t>()); break;
                default: launch_pdl(k_conv_mac_small<1>, dim3(gs), dim3(128), sm, c.stream, tt.c_(), colp, no, C, W, k, F, dwb.get(), bpow, dbq.get(), mask_pt, nl, N, c.primes, yp.as<uint64_t>()); break;
            }
            check_launch("k_conv_mac_small");
        } else {
        switch (FG) {
            case 8: launch_pdl(k_conv_mac<8>, dim3(grid), dim3(128), 0, c.stream, tt.c_(), colp, no, C, W, k, F, dwq.get(), dbq.get(), mask_pt, nl, N, c.primes, yp.as<uint64_t>()); break;
            case 4: launch_pdl(k_conv_mac<4>, dim3(grid), dim3(128), 0, c.stream, tt.c_(), colp, no, C, W, k, F, dwq.get(), dbq.get(), mask_pt, nl, N, c.primes, yp.as<uint64_t>()); break;
            case 2: launch_pdl(k_conv_mac<2>, dim3(grid), dim3(128), 0, c.stream, tt.c_(), colp, no, C, W, k, F, dwq.get(), dbq.get(), mask_pt, nl, N, c.primes, yp.as<uint64_t>()); break;
            default: launch_pdl(k_conv_mac<1>, dim3(grid), dim3(128), 0, c.stream, tt.c_(), colp, no, C, W, k, F, dwq.get(), dbq.get(), mask_pt, nl, N, c.primes, yp.as<uint64_t>()); break;
        }
        check_launch("k_conv_mac");
        }
        std::vector<const uint64_t *> ins((size_t)F * no);
        std::vector<const uint64_t *> outs((size_t)F * no);
        for (int f = 0; f < F; f++)
            for (int o = 0; o < no; o++) {
                ins[(size_t)f * no + o] = yp.as<uint64_t>() + ((size_t)f * no + o) * ctw;
                outs[(size_t)f * no + o] = Y[(size_t)f * nout + o0 + o];
            }
        PtrTable ti(c, ins), to(c, outs);
        rescale(c, ti.c_(), to.m_(), F * no, 2, level);
    }
}

// oracle/ckks_oracle.c:orc_poly_activation -- one relinearisation (two if c3 != 0) and the
// c1*x term folded into the final rescale.
static void poly_activation_chunk(Ctx &c, const uint64_t *const *X, int count, int level, const int64_t *kc, int c3_zero,
                                  uint64_t *const *Out) {
    const int N = c.n;
    const size_t w1 = (size_t)2 * level * N;
    Scratch x2(c, sizeof(uint64_t) * count * w1), pre(c, sizeof(uint64_t) * count * w1);
    PtrTable tx2(c, strided(x2.as<uint64_t>(), count, w1)), tpre(c, strided(pre.as<uint64_t>(), count, w1));
    mul_batch(c, X, X, tx2.m_(), count, level);  // x^2 at level-1
    if (c3_zero) {
        scale_axpy(c, tx2.c_(), X, tpre.m_(), count, 2, level, level + 1, limb_scalars(c, kc[1], level),
                   limb_scalars(c, kc[2], level));
        rescale(c, tpre.c_(), Out, count, 2, level - 1);
    } else {
        Scratch inner(c, sizeof(uint64_t) * count * w1), xs(c, sizeof(uint64_t) * count * 2 * (level + 1) * N),
            d3(c, sizeof(uint64_t) * count * 3 * level * N);
        PtrTable tin(c, strided(inner.as<uint64_t>(), count, w1)),
            txs(c, strided(xs.as<uint64_t>(), count, (size_t)2 * (level + 1) * N)),
            td3(c, strided(d3.as<uint64_t>(), count, (size_t)3 * level * N));
        mul_scalar(c, X, txs.m_(), count, 2, level + 1, limb_scalars(c, kc[0], level + 1));
        rescale(c, txs.c_(), tin.m_(), count, 2, level);
        add_const(c, tin.m_(), count, level, limb_scalars(c, kc[1], level));
        tensor(c, tx2.c_(), tin.c_(), td3.m_(), count, level);
        // x' k1 joins (d0, d1) before the fused relinearise + rescale
        axpy(c, td3.m_(), X, count, 2, level, level + 1, limb_scalars(c, kc[2], level));
        relin_rescale_batch(c, td3.c_(), Out, count, level - 1);
    }
    add_const(c, Out, count, level - 1, limb_scalars(c, kc[3], level - 1));
}

void poly_activation(Ctx &c, const uint64_t *const *X, int count, int level, const int64_t *kc, int c3_zero,
                     uint64_t *const *Out) {
    if (level < 2) throw VrError(3, "poly_activation needs two levels");
    // scratch per ciphertext is dominated by the relinearisation ModUp (nl * (nl+1) * N words)
    const size_t per_ct = sizeof(uint64_t) * (size_t)c.n * ((size_t)(level + 1) * (level + 2) + 12 * (level + 1));
    const int chunk = (int)std::max<size_t>(1, std::min<size_t>((size_t)count, ((size_t)4 << 30) / per_ct));
    for (int c0 = 0; c0 < count; c0 += chunk) {
        const int n = std::min(chunk, count - c0);
        poly_activation_chunk(c, X + c0, n, level, kc, c3_zero, Out + c0);
    }
}

template <int UG, int JU>
static void pt_matvec_ug(Ctx &c, const uint64_t *const *X, int nx, const uint64_t *const *PT, int ny, int level,
                         uint64_t *const *Y) {
    const int N = c.n, nl = level + 1;
    const size_t ctw = (size_t)2 * nl * N;
    const int chunk = (int)std::max<size_t>(UG, std::min<size_t>((size_t)ny, ((size_t)2 << 30) / (ctw * 8)));
    Scratch yp(c, sizeof(uint64_t) * (size_t)std::min(chunk, ny) * ctw);
    for (int u0 = 0; u0 < ny; u0 += chunk) {
        const int nu = std::min(chunk, ny - u0);
        dim3 grid(nblocks(N / 2, 128), nl, (nu + UG - 1) / UG);
        launch_pdl(k_pt_matvec<UG, JU>, dim3(grid), dim3(128), 0, c.stream, X, nx, PT + (size_t)u0 * nx, nu, nl, N, c.primes, yp.as<uint64_t>());
        check_launch("k_pt_matvec");
        std::vector<const uint64_t *> ins(nu);
        for (int u = 0; u < nu; u++) ins[u] = yp.as<uint64_t>() + (size_t)u * ctw;
        PtrTable ti(c, ins);
        rescale(c, ti.c_(), Y + u0, nu, 2, level);
    }
}

void pt_matvec(Ctx &c, const uint64_t *const *X, int nx, const uint64_t *const *PT, int ny, int level, uint64_t *const *Y) {
    static const int ug = [] {
        const char *e = getenv("VR_PMV_UG");
        return e ? atoi(e) : 2;
    }();
    switch (ug) {
        case 1: pt_matvec_ug<1, 4>(c, X, nx, PT, ny, level, Y); break;
        case 3: pt_matvec_ug<2, 4>(c, X, nx, PT, ny, level, Y); break;
        case 4: pt_matvec_ug<4, 2>(c, X, nx, PT, ny, level, Y); break;
        default: pt_matvec_ug<2, 2>(c, X, nx, PT, ny, level, Y); break;
    }
}

}  // namespace vr
