/*
 * vrhe.h -- C-ABI of libvrhe.so, the B200-native RNS-CKKS evaluator behind the
 * packedhe SlotEngine surface (arXiv 2512.18646, Volley Revolver Inference++).
 *
 * The reference has no native code; its "FFI" for this path is the Python
 * method surface of SlotEngine (/root/reference/pkg/src/packedhe/engine.py)
 * and the multi-ciphertext drivers (multicipher.py, pipeline.py).  Each entry
 * point below names the reference call it replaces.  INTEGRATION.md shows the
 * ctypes binding a packedhe maintainer would add.
 *
 * Conventions
 *   - All `uint64_t *` ciphertext/plaintext arguments are DEVICE pointers.
 *     A ciphertext at level l with degree d is [d+1][l+1][N] uint64 residues in
 *     NTT form (limb i is mod primes[i]); a plaintext is [l+1][N].
 *   - Pointer-table arguments (`const uint64_t *const *`) are HOST arrays of
 *     device pointers, one entry per ciphertext in the batch.
 *   - Every call is stream-ordered on the stream given to vr_set_stream and
 *     returns a status: VR_OK, or an error whose message vr_last_error()
 *     returns.  The Python host layer maps codes to the reference exception
 *     classes (CapacityError / LayoutError / EngineError, engine.py:32-41).
 */
#ifndef VRHE_H
#define VRHE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VR_OK 0
#define VR_ERR_CAPACITY 1 /* engine.py:36-37 CapacityError */
#define VR_ERR_LAYOUT 2   /* engine.py:40-41 LayoutError */
#define VR_ERR_ENGINE 3   /* engine.py:32-33 EngineError */
#define VR_ERR_CUDA 4

typedef struct vr_ctx vr_ctx;
/* a ciphertext owned through the C-ABI (engine.py:140-150): device residues + level/degree/scale */
typedef struct vr_ct vr_ct;

/* ---- context ------------------------------------------------------------- */
/* EngineParams + SlotEngine.__init__ (engine.py:54-90, 175-178).  primes holds
 * num_q ciphertext primes q0..q_{num_q-1} followed by the special prime P.
 * Generates the secret and public key on the device from `seed`. */
int vr_ctx_create(int log_n, int num_q, const uint64_t *primes, uint64_t seed, int sym_enc, int device, vr_ctx **out);
int vr_ctx_destroy(vr_ctx *ctx);
const char *vr_last_error(void);
/* total kernels this library has launched (instrumentation for bench.py) */
unsigned long long vr_launch_count(void);
/* order every later call on cuda_stream (NULL = the legacy default stream); the context's
 * private stream (the default after vr_ctx_create) stays alive until vr_ctx_destroy */
int vr_set_stream(vr_ctx *ctx, void *cuda_stream);
/* `stream` first waits for everything queued on the context's stream, then becomes the context's
 * stream (vr_set_stream switches back): runs the following calls on a side stream, e.g. the deferred
 * encryption of a product's operands (multicipher.py:62-85) on the slot stream of that product */
int vr_fork_stream(vr_ctx *ctx, void *stream);
int vr_sync(vr_ctx *ctx);

/* ---- ciphertexts owned through the C-ABI (host-buffer I/O, no PyTorch) -------- */
/* Ciphertext objects for bindings that own no device memory (cgo / JNI / plain ctypes): the
 * SlotEngine.enc -> ops -> dec round trip of engine.py:193-206 from host buffers.  vr_ct_data is a
 * device pointer accepted by every raw entry point below. */
int vr_ct_alloc(vr_ctx *ctx, int level, int degree, double scale, vr_ct **out);
int vr_ct_free(vr_ctx *ctx, vr_ct *ct);
uint64_t *vr_ct_data(const vr_ct *ct);
int vr_ct_level(const vr_ct *ct);
int vr_ct_degree(const vr_ct *ct);
double vr_ct_scale(const vr_ct *ct);
/* residues [degree+1][level+1][N] (uint64, limb-major, NTT form) to / from host memory */
int vr_ct_upload(vr_ctx *ctx, vr_ct *ct, const uint64_t *host);
int vr_ct_download(vr_ctx *ctx, const vr_ct *ct, uint64_t *host);
/* SlotEngine.enc (engine.py:193-202) from host doubles [count][nvals] into fresh top-level cts */
int vr_encrypt_host(vr_ctx *ctx, const double *host_vals, int count, int nvals, double scale, uint64_t nonce0,
                    vr_ct *const *cts);
/* SlotEngine.dec (engine.py:204-206) of count cts into host doubles [count][S] */
int vr_decrypt_host(vr_ctx *ctx, const vr_ct *const *cts, int count, double *host_out);
/* matmul_outer (multicipher.py:88-103) on vr_ct operands: out[b] (degree 1, level - 1) receives
 * rescale(relin(sum_k L[b*n+k] (x) R[k])) and the scale L.scale * R.scale / q_level */
int vr_matmul_outer_ct(vr_ctx *ctx, const vr_ct *const *L, const vr_ct *const *R, int n, int nb, vr_ct *const *out);

/* ---- multi-GPU: native NCCL communicator per context ------ */
/* 128-byte NCCL unique id, generated on one rank and shared with the others (any channel) */
int vr_comm_unique_id(void *id_out);
int vr_comm_init(vr_ctx *ctx, const void *id, int rank, int nranks);
int vr_comm_destroy(vr_ctx *ctx);
/* sum degree-2 partials [polys][level+1][N] over the ranks (uint64 NCCL sum, <= 8 ranks) and reduce
 * mod q_i: root < 0 = all-reduce (every rank gets the sum), else only rank `root` (multicipher.py:100-102) */
int vr_sum_partials(vr_ctx *ctx, uint64_t *data, long long polys, int level, int root);

/* ---- keys ---------------------------------------------------------------- */
int vr_gen_relin_key(vr_ctx *ctx);
/* Galois element 5^(steps mod S) mod 2N for a LEFT rotation (engine.py:232-236) */
int vr_galois_elt(vr_ctx *ctx, int64_t steps, uint32_t *g_out);
int vr_gen_galois_key(vr_ctx *ctx, uint32_t g);
/* host-buffer exports for parity tests: s in NTT form [np][N]; pk [2][L+1][N];
 * switching keys [L+1][2][np][N] */
int vr_export_secret(vr_ctx *ctx, uint64_t *host_out);
int vr_export_public_key(vr_ctx *ctx, uint64_t *host_out);
int vr_export_relin_key(vr_ctx *ctx, uint64_t *host_out);
int vr_export_galois_key(vr_ctx *ctx, uint32_t g, uint64_t *host_out);

/* ---- transforms ---------------------------------------------------------- */
/* in-place NTT/INTT of [polys][limbs][N] (limb i uses prime index prime0 + i) */
int vr_ntt(vr_ctx *ctx, uint64_t *data, int polys, int limbs, int prime0, int inverse);

/* ---- encode / encrypt / decrypt -- SlotEngine.enc / dec / mask ----------- */
/* SlotEngine.mask + plaintext encoding (engine.py:244-251): values [count][nvals]
 * (device doubles, zero-padded to S slots) -> plaintexts [count][level+1][N] */
int vr_encode(vr_ctx *ctx, const double *vals, int count, int nvals, int level, double scale, uint64_t *pt_out);
/* integer coefficients of the encoding (test hook), m_out [count][N] int64 */
int vr_encode_coeffs(vr_ctx *ctx, const double *vals, int count, int nvals, double scale, int64_t *m_out);
/* SlotEngine.enc (engine.py:193-202): fresh encryption, ciphertext c uses nonce0+c */
int vr_encrypt(vr_ctx *ctx, const double *vals, int count, int nvals, int level, double scale, uint64_t nonce0,
               uint64_t *ct_out);
/* encode_left / encode_right / encode_image_columns (multicipher.py:62-120) without host-side
 * broadcasting: ciphertext c encrypts slot values src[c*sc + (j/p)*s1 + (j%p)*s2] for j < nvals
 * (zeros beyond), src = the raw device matrix/images */
int vr_encrypt_strided(vr_ctx *ctx, const double *src, long long sc, long long s1, long long s2, int p, int nvals, int count,
                       int level, double scale, uint64_t nonce0, uint64_t *ct_out);
/* encode_left + encode_right of one product (multicipher.py:62-85) as one launch: ciphertexts
 * 0..count0-1 from (src0, strides 0) into ct0, then count1 from (src1, strides 1) into ct1, nonces
 * nonce0 + c consecutive over both (secret-key encryption only) */
int vr_encrypt_strided2(vr_ctx *ctx, const double *src0, long long sc0, long long s1_0, long long s2_0, int p0, int nvals0,
                        int count0, uint64_t *ct0, const double *src1, long long sc1, long long s1_1, long long s2_1, int p1,
                        int nvals1, int count1, uint64_t *ct1, int level, double scale, uint64_t nonce0);
/* The same strided encryptions from HOST arrays (the raw matrices encode_left / encode_right /
 * encode_image_columns receive, multicipher.py:62-85,106-120): host[0..len) is staged through the
 * context's pinned ring into stream-ordered device scratch; the source of ciphertext c starts at
 * element off + c*sc.  The host array may be reused as soon as the call returns. */
int vr_encrypt_strided_host(vr_ctx *ctx, const double *host, long long len, long long off, long long sc, long long s1,
                            long long s2, int p, int nvals, int count, int level, double scale, uint64_t nonce0,
                            uint64_t *ct_out);
int vr_encrypt_strided2_host(vr_ctx *ctx, const double *host0, long long len0, long long off0, long long sc0, long long s1_0,
                             long long s2_0, int p0, int nvals0, int count0, uint64_t *ct0, const double *host1,
                             long long len1, long long off1, long long sc1, long long s1_1, long long s2_1, int p1, int nvals1,
                             int count1, uint64_t *ct1, int level, double scale, uint64_t nonce0);
/* SlotEngine.dec (engine.py:204-206) to host memory without blocking the caller: decrypt + decode
 * on `stream` (NULL: the context stream; e.g. the slot stream that produced the ciphertexts), copy
 * the [count][S] real slots into a pinned buffer owned by the context and record an event.
 * vr_decode_wait(ticket) blocks until that event, copies the slots to host_out ([count][S] doubles,
 * may be NULL) and releases the ticket.  Lets a caller keep encrypt -> product -> decode steps in flight. */
int vr_decode_submit(vr_ctx *ctx, const uint64_t *const *cts, const int *degs, const int *levels, const double *scales,
                     int count, void *stream, int *ticket);
int vr_decode_wait(vr_ctx *ctx, int ticket, double *host_out);
/* SlotEngine.dec (engine.py:204-206): decrypt on q0 and decode to real slots.
 * out: device [count][S] doubles (may be NULL); coeffs_out: device [count][N] int64 (may be NULL). */
int vr_decrypt_decode(vr_ctx *ctx, const uint64_t *const *cts, const int *degs, const int *levels, const double *scales,
                      int count, double *out, int64_t *coeffs_out);

/* ---- primitive arithmetic (batched) ------------------------------------- */
/* SlotEngine.add (engine.py:208-213); op 0 = add, 1 = sub */
int vr_add(vr_ctx *ctx, const uint64_t *const *a, const uint64_t *const *b, uint64_t *const *out, int count, int deg,
           int level, int op);
int vr_tensor(vr_ctx *ctx, const uint64_t *const *a, const uint64_t *const *b, uint64_t *const *out, int count, int level);
int vr_relin(vr_ctx *ctx, const uint64_t *const *d3, uint64_t *const *out, int count, int level);
int vr_rescale(vr_ctx *ctx, const uint64_t *const *in, uint64_t *const *out, int count, int deg, int level);
/* relinearise + rescale as one rounding step, (P d + KS) / (P q_l): degree 2 at level -> degree 1 at level-1 */
int vr_relin_rescale(vr_ctx *ctx, const uint64_t *const *d3, uint64_t *const *out, int count, int level);
/* SlotEngine.mul (engine.py:215-220): tensor -> relinearise -> rescale */
int vr_mul(vr_ctx *ctx, const uint64_t *const *a, const uint64_t *const *b, uint64_t *const *out, int count, int level);
/* SlotEngine.cmul (engine.py:222-230) building blocks: plaintext / integer-scalar products */
int vr_mul_plain(vr_ctx *ctx, const uint64_t *const *ct, const uint64_t *const *pt, uint64_t *const *out, int count, int deg,
                 int level, int shared_pt);
int vr_mul_scalar(vr_ctx *ctx, const uint64_t *const *ct, int64_t s, uint64_t *const *out, int count, int deg, int level);
int vr_add_const(vr_ctx *ctx, uint64_t *const *ct, int64_t s, int count, int level);
int vr_drop_level(vr_ctx *ctx, const uint64_t *const *in, uint64_t *const *out, int count, int deg, int level_from,
                  int level_to);
/* SlotEngine.rot (engine.py:232-236), hoisted: out[c*nrot + r] = rot(in[c], steps[r]) */
int vr_rotate(vr_ctx *ctx, const uint64_t *const *in, uint64_t *const *out, int count, int level, int nrot,
              const int64_t *steps);
/* raw key switch of one polynomial [level+1][N] with the relin key (g == 0) or Galois key g; out [2][level+1][N] */
int vr_keyswitch(vr_ctx *ctx, const uint64_t *poly, int level, uint32_t g, uint64_t *out);
/* integer-pipe roofline probe: blocks x 256 threads x iters x 8 register-only NTT butterflies */
int vr_bench_butterflies(vr_ctx *ctx, int blocks, int iters, uint64_t *d_sink);
/* FP64-pipe roofline probe (the FP64 NTT butterfly for primes < 2^46): blocks x 256 threads x iters x 64 butterflies */
int vr_bench_butterflies_f64(vr_ctx *ctx, int blocks, int iters, uint64_t *d_sink);
/* reduce residue sums (< 2^64) mod q_i in place: [polys][level+1][N] (after an NCCL uint64 sum) */
int vr_mod_reduce(vr_ctx *ctx, uint64_t *data, long long polys, int level);

/* ---- column-ciphertext drivers ------------------------------------------ */
/* matmul_outer (multicipher.py:88-103): out[b] = rescale(relin(sum_k L[b*n+k] (x) R[k])), nb row
 * blocks share R (nb in {1,2,4}) */
int vr_matmul_outer(vr_ctx *ctx, const uint64_t *const *L, const uint64_t *const *R, int n, int nb, int level,
                    uint64_t *const *out);
/* `count` independent matmul_outer products (multicipher.py:88-103 once per operand pair) in one launch
 * sequence: out[b] = rescale(relin(sum_k L[b*n+k] (x) R[b*n+k])), all operands at `level`.  Residues
 * equal those of `count` separate vr_matmul_outer calls; small products share six kernel launches. */
int vr_matmul_outer_many(vr_ctx *ctx, const uint64_t *const *L, const uint64_t *const *R, int n, int count, int level,
                         uint64_t *const *out);
/* matmul_outer without waiting for the result: the product is computed on one of the context's
 * slot streams, which first waits for all work already queued on the context stream.  *slot_stream
 * receives that stream (the result is complete once it reaches the current point of that stream),
 * or NULL if the call ran synchronously on the context stream.  Consecutive independent calls
 * overlap on the device.  The caller must order every later use of `out` (and every reuse of the
 * operand buffers) after *slot_stream, e.g. with vr_join. */
int vr_matmul_outer_async(vr_ctx *ctx, const uint64_t *const *L, const uint64_t *const *R, int n, int nb, int level,
                          uint64_t *const *out, void **slot_stream);
/* the slot stream the next vr_matmul_outer_async call will run on (allocate its output there) */
int vr_async_slot(vr_ctx *ctx, void **slot_stream);
/* make the context stream wait for everything queued on the slot streams */
int vr_join(vr_ctx *ctx);
/* the degree-2 partial sum only (multi-GPU: all-reduce, vr_mod_reduce, then vr_relin + vr_rescale) */
int vr_tensor_sum(vr_ctx *ctx, const uint64_t *const *L, const uint64_t *const *R, int n, int nb, int level,
                  uint64_t *const *out);
/* the two halves matmul_outer overlaps: mode 1 writes d2 = sum L1 R1 (poly 2 of out), mode 2 writes
 * (d0, d1) (polys 0, 1 of out); out is one [3][level+1][N] buffer */
int vr_tensor_sum_mode(vr_ctx *ctx, const uint64_t *const *L, const uint64_t *const *R, int n, int level, uint64_t *out, int mode);
/* conv_columns (multicipher.py:123-162) for C channels x F filters:
 *   Y[f*nout+o] = rescale(mask * (sum_{c,q,p} w[f][c][p][q] * rot(X[c*W + cols[o]+q], p) + bias[f]))
 * w: host int64 [F][C][k][k] (quantised weights), bias_res: host [F][level+1] residues of the bias
 * integer (it may exceed 64 bits), mask: device plaintext [level+1][N] */
int vr_conv_columns(vr_ctx *ctx, const uint64_t *const *X, int C, int W, int k, const int64_t *w, const uint64_t *bias_res, int F,
                    const int *out_cols, int nout, const uint64_t *mask_pt, int level, uint64_t *const *Y);
/* plaintext-weight dense layer on column ciphertexts (config 3; built from SlotEngine.cmul + add,
 * engine.py:208-230): Y[u] = rescale(sum_j PT[u*nx + j] (.) X[j]), PT are encoded plaintexts [level+1][N] */
int vr_pt_matvec(vr_ctx *ctx, const uint64_t *const *X, int nx, const uint64_t *const *PT, int ny, int level,
                 uint64_t *const *Y);
/* poly_activation (pipeline.py:180-197) on a batch; kc = integer constants {c3, c2, c1, c0} at their
 * target scales */
int vr_poly_activation(vr_ctx *ctx, const uint64_t *const *x, int count, int level, const int64_t *kc, int c3_zero,
                       uint64_t *const *out);

#ifdef __cplusplus
}
#endif

#endif /* VRHE_H */
