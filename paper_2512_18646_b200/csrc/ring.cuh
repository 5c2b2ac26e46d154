// ring.cuh -- device-level building blocks shared by abi.cu and the drivers.
// All pointer-table arguments are DEVICE arrays of device pointers; each entry
// addresses one ciphertext laid out [poly][limb][N] (limb i uses prime i).
#pragma once
#include "vrhe_internal.cuh"

namespace vr {

struct LimbScalars {
    uint64_t v[MAXP], sh[MAXP];
};
LimbScalars limb_scalars(const Ctx &c, int64_t s, int nl);

// elementwise (op 0 = add, 1 = sub)
void binop(Ctx &c, const uint64_t *const *A, const uint64_t *const *B, uint64_t *const *O, int count, int polys, int nl, int op);
void tensor(Ctx &c, const uint64_t *const *A, const uint64_t *const *B, uint64_t *const *O, int count, int nl);
void mul_plain(Ctx &c, const uint64_t *const *C, const uint64_t *const *P, uint64_t *const *O, int count, int polys, int nl,
               int shared_pt);
void mul_scalar(Ctx &c, const uint64_t *const *C, uint64_t *const *O, int count, int polys, int nl, const LimbScalars &s);
void add_const(Ctx &c, uint64_t *const *C, int count, int nl, const LimbScalars &s);
// O[c][p][i] += B[c][p][i] * s_i for i < nl (B has nlb >= nl limbs per poly)
void axpy(Ctx &c, uint64_t *const *O, const uint64_t *const *B, int count, int polys, int nl, int nlb, const LimbScalars &s);
// O = C * s + B * t per limb (B with nlb >= nl limbs): one pass instead of mul_scalar + axpy
void scale_axpy(Ctx &c, const uint64_t *const *C, const uint64_t *const *B, uint64_t *const *O, int count, int polys, int nl,
                int nlb, const LimbScalars &s, const LimbScalars &t);
void permute(Ctx &c, const uint64_t *const *C, uint64_t *const *O, int count, int polys, int nl, uint32_t g);
void copy_limbs(Ctx &c, const uint64_t *const *C, uint64_t *const *O, int count, int polys, int nl_in, int nl_out, int limb0);
void mod_fixup(Ctx &c, uint64_t *data, long long count_polys, int nl);
void bfly_peak(Ctx &c, int blocks, int iters, uint64_t *sink);
void bfly_peak_f64(Ctx &c, int blocks, int iters, uint64_t *sink);  // iters x 64 butterflies per thread
// mode 1: d2 only, mode 2: (d0, d1) only (single row block)
void tensor_sum_mode(Ctx &c, const uint64_t *const *L, const uint64_t *const *R, int n, int nb, int nl, uint64_t *const *O,
                     int mode);
void tensor_sum(Ctx &c, const uint64_t *const *L, const uint64_t *const *R, int n, int nb, int nl, uint64_t *const *O);
bool tensor_sum_takes_params(int nb);
// B independent products in one launch: O[b] = sum_k L[b*n + k] (x) R[b*n + k]
void tensor_sum_many(Ctx &c, const uint64_t *const *L, const uint64_t *const *R, int n, int B, int nl, uint64_t *const *O);

// rescale: in [polys][l+1][N] -> out [polys][l][N] for each ciphertext
void rescale(Ctx &c, const uint64_t *const *In, uint64_t *const *Out, int count, int polys, int level);

// Key switching.  ModUp of `count` polys (each [l+1][N], NTT) into
// D [count][l+1][l+2][N] (NTT form; target l+1 is the special prime; the
// digit's own prime is not materialised -- the inner product reads it from
// the input polynomial).
void modup(Ctx &c, const uint64_t *const *Polys, int count, int level, uint64_t *D);
// Full key switch of `count` polys with `key` ([L+1][2][np][N]) into Out[c] = [2][l+1][N].
void keyswitch_poly(Ctx &c, const uint64_t *const *Polys, int count, int level, const uint64_t *key, uint64_t *const *Out);

// Convenience wrappers operating on pointer tables (device) of ciphertexts.
void relin_batch(Ctx &c, const uint64_t *const *D3, uint64_t *const *Out, int count, int level);  // deg2 -> deg1, same level
// deg2 at level l -> deg1 at level l-1: (P d + KS-acc) / (P q_l) in one rounding step
// d01_ready: event after which (d0, d1) of D3 are valid (they may be computed on another stream while
// the key switch of d2 runs); nullptr if they are already ordered on c.stream
void relin_rescale_batch(Ctx &c, const uint64_t *const *D3, uint64_t *const *Out, int count, int level,
                         cudaEvent_t d01_ready = nullptr);
void rotate_batch(Ctx &c, const uint64_t *const *In, uint64_t *const *Out, int count, int level, int nrot, const uint32_t *gs);

uint64_t *galois_key(Ctx &c, uint32_t g);
uint64_t *relin_key(Ctx &c);

// host helper: device pointer table (cached by value in the context)
struct PtrTable {
    const void *const *p;
    PtrTable(Ctx &c, const std::vector<const uint64_t *> &v)
        : p(cached_table(c, (const void *const *)v.data(), v.size())) {}
    const uint64_t *const *c_() const { return (const uint64_t *const *)p; }
    uint64_t *const *m_() const { return (uint64_t *const *)p; }
};

}  // namespace vr
