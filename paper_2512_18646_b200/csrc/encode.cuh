// encode.cuh -- encode / encrypt / decrypt / keygen entry points (device level).
#pragma once
#include "ring.cuh"

namespace vr {

void encode_coeffs(Ctx &c, const double *d_vals, int count, int nvals, double scale, int64_t *d_m);
void encode_plain(Ctx &c, const double *d_vals, int count, int nvals, int level, double scale, uint64_t *d_pt);
void encrypt(Ctx &c, const double *d_vals, int count, int nvals, int level, double scale, uint64_t nonce0, uint64_t *d_ct);
// ciphertext c encrypts slot values src[c*sc + (j/p)*s1 + (j%p)*s2], j < nvals (zeros beyond)
void encrypt_src2(Ctx &c, const double *src0, long long sc0, long long s1_0, long long s2_0, int p0, int nvals0, int count0,
                  uint64_t *d_ct0, const double *src1, long long sc1, long long s1_1, long long s2_1, int p1, int nvals1,
                  int count1, uint64_t *d_ct1, int level, double scale, uint64_t nonce0);
void encrypt_src(Ctx &c, const double *src, long long sc, long long s1, long long s2, int p, int nvals, int count, int level,
                 double scale, uint64_t nonce0, uint64_t *d_ct);
void decrypt_decode(Ctx &c, const uint64_t *const *d_cts, const int *d_degs, const int *d_levels, const double *d_scales,
                    int count, double *d_out, int64_t *d_coeffs_out);
void keygen(Ctx &c);

// drivers (drivers.cu)
void mul_batch(Ctx &c, const uint64_t *const *A, const uint64_t *const *B, uint64_t *const *Out, int count, int level);
// comm.cu: NCCL communicator of the context and the partial-product sum of config 5a
void comm_unique_id(void *out128);
void comm_init(Ctx &c, const void *id, int rank, int nranks);
void comm_destroy(Ctx &c);
void sum_partials(Ctx &c, uint64_t *data, long long polys, int level, int root);
// one_pass: one (d0, d1, d2) tensor-sum pass then the key-switch chain, all on c.stream (the form
// recorded into the asynchronous per-slot graphs, graph.cu)
void matmul_outer(Ctx &c, const uint64_t *const *L, const uint64_t *const *R, int n, int nb, int level, uint64_t *const *Out,
                  bool one_pass = false);
void matmul_outer_many(Ctx &c, const uint64_t *const *L, const uint64_t *const *R, int n, int B, int level, uint64_t *const *Out);
void conv_columns(Ctx &c, const std::vector<const uint64_t *> &X, int C, int W, int k, const int64_t *w, const uint64_t *bias,
                  int F, const int *out_cols, int nout, const uint64_t *mask_pt, int level, const std::vector<uint64_t *> &Y);
void pt_matvec(Ctx &c, const uint64_t *const *X, int nx, const uint64_t *const *PT, int ny, int level, uint64_t *const *Y);
void poly_activation(Ctx &c, const uint64_t *const *X, int count, int level, const int64_t *kc, int c3_zero,
                     uint64_t *const *Out);

}  // namespace vr
