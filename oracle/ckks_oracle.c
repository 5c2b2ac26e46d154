/*
 * ckks_oracle.c -- CPU RNS-CKKS restatement used as the RESIDUE ORACLE.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package
 * (paper_2512_18646_b200/) links, loads or calls this file.  Only tests/,
 * __graft_entry__.smoke() and bench.py (cpu_baseline leg / --impl reference)
 * use it, and there only as the checker or as the timed CPU baseline.
 *
 * What it restates.  The reference (packedhe, /root/reference/pkg) is an
 * exact float64 slot simulator: SlotEngine.enc/dec/add/mul/cmul/rot
 * (engine.py:193-251) with no ring arithmetic at all (engine.py:1-9,
 * SPEC.md:7).  The north star asks for real RNS-CKKS behind that surface, so
 * this file is the *definition* of every residue the GPU must reproduce
 * bit-for-bit ("parity unpinned" against the reference at residue level --
 * the reference has no residues; decoded values are pinned against the
 * reference simulator in tests/).  Slot semantics follow the reference:
 *   - enc zero-pads into the leading slots            engine.py:193-202
 *   - rot(l) is a cyclic LEFT rotation (np.roll(-l))   engine.py:232-236
 *   - mul/cmul consume one level (depth+1)             engine.py:215-230
 * and the fused drivers restate the op order of
 *   - matmul_outer        multicipher.py:88-103
 *   - conv_columns        multicipher.py:123-162
 *   - poly_activation     pipeline.py:180-197
 *
 * Everything is integer-exact except encode/decode, whose double-precision
 * FFT is written with an explicit operation order and compiled with
 * -ffp-contract=off so the GPU (which uses __dmul_rn/__dadd_rn) produces
 * identical doubles and therefore identical rounded coefficients.
 *
 * Conventions (shared with the CUDA library):
 *   ciphertext at level l = [deg+1][l+1][N] uint64, NTT domain, limb-major;
 *   primes q[0..L] ciphertext chain, q[L+1] = special prime P;
 *   NTT = Cooley-Tukey negacyclic, natural in -> bit-reversed out
 *         (a_hat[k] = a(psi^(2*br(k)+1))), INTT = Gentleman-Sande inverse.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

#define ORC_MAXP 40
#define CDT_LEN 32

/* ------------------------------------------------------------------ */
/* scalar modular arithmetic (obviously-correct u128 versions)          */
/* ------------------------------------------------------------------ */
static inline uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a * b) % q); }
static inline uint64_t addmod(uint64_t a, uint64_t b, uint64_t q) { uint64_t s = a + b; return s >= q ? s - q : s; }
static inline uint64_t submod(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }
static uint64_t powmod(uint64_t b, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = mulmod(r, b, q);
        b = mulmod(b, b, q);
        e >>= 1;
    }
    return r;
}
static inline uint64_t invmod(uint64_t a, uint64_t q) { return powmod(a, q - 2, q); }
/* signed 64-bit integer -> [0,q) */
static inline uint64_t reduce_i64(int64_t v, uint64_t q) {
    if (v >= 0) return (uint64_t)v % q;
    uint64_t r = ((uint64_t)(-(v + 1)) + 1) % q; /* |v| mod q without overflow */
    return r ? q - r : 0;
}
/* centered lift of x in [0,from) into Z_to (x > from/2 is read as x - from) */
static inline uint64_t lift_centered(uint64_t x, uint64_t from, uint64_t to) {
    if (x > (from >> 1)) {
        uint64_t r = (from - x) % to;
        return r ? to - r : 0;
    }
    return x % to;
}

/* ------------------------------------------------------------------ */
/* primes                                                              */
/* ------------------------------------------------------------------ */
static int is_prime_u64(uint64_t n) {
    if (n < 2) return 0;
    static const uint64_t small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (int i = 0; i < 12; i++) {
        if (n == small[i]) return 1;
        if (n % small[i] == 0) return 0;
    }
    uint64_t d = n - 1;
    int r = 0;
    while ((d & 1) == 0) { d >>= 1; r++; }
    for (int i = 0; i < 12; i++) {
        uint64_t x = powmod(small[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int comp = 1;
        for (int j = 1; j < r; j++) {
            x = mulmod(x, x, n);
            if (x == n - 1) { comp = 0; break; }
        }
        if (comp) return 0;
    }
    return 1;
}

/* Prime chain: for each requested bit size (in order) the largest prime
 * p < 2^bits with p == 1 (mod 2N) not already taken.  Returns 0 on success. */
int orc_gen_primes(int log_n, int count, const int *bits, uint64_t *out) {
    uint64_t two_n = 2ull << log_n;
    for (int i = 0; i < count; i++) {
        if (bits[i] < log_n + 2 || bits[i] > 61) return -1;
        uint64_t top = (bits[i] == 64) ? ~0ull : ((1ull << bits[i]) - 1);
        uint64_t c = (top / two_n) * two_n + 1;
        if (c > top) c -= two_n;
        for (;;) {
            if (c < two_n) return -2;
            int used = 0;
            for (int j = 0; j < i; j++) used |= (out[j] == c);
            if (!used && is_prime_u64(c)) break;
            c -= two_n;
        }
        out[i] = c;
    }
    return 0;
}

/* minimal primitive 2N-th root of unity mod q */
static uint64_t min_psi(uint64_t q, int n) {
    uint64_t two_n = 2ull * n, psi = 0;
    for (uint64_t g = 2;; g++) {
        uint64_t x = powmod(g, (q - 1) / two_n, q);
        if (powmod(x, n, q) == q - 1) { psi = x; break; }
    }
    uint64_t best = psi, sq = mulmod(psi, psi, q), cur = psi;
    for (int k = 1; k < n; k++) { /* odd powers psi^(2k+1) */
        cur = mulmod(cur, sq, q);
        if (cur < best) best = cur;
    }
    return best;
}

static inline uint32_t bitrev(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

/* ------------------------------------------------------------------ */
/* counter-based RNG (SplitMix64 finaliser) + samplers                 */
/* ------------------------------------------------------------------ */
enum {
    DOM_SK = 1, DOM_PK_A = 2, DOM_PK_E = 3, DOM_RLK_A = 4, DOM_RLK_E = 5,
    DOM_GAL_A = 6, DOM_GAL_E = 7, DOM_ENC_V = 8, DOM_ENC_E0 = 9, DOM_ENC_E1 = 10,
    DOM_ENC_A = 11
};
static inline uint64_t fmix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
uint64_t orc_stream_key(uint64_t seed, uint64_t dom, uint64_t a, uint64_t b) {
    uint64_t k = fmix64(seed ^ (dom * 0x9E3779B97F4A7C15ull));
    k = fmix64(k ^ (a * 0xC2B2AE3D27D4EB4Full));
    k = fmix64(k ^ (b * 0x165667B19E3779F9ull));
    return k;
}
static inline uint64_t rnd(uint64_t key, uint64_t i) { return fmix64(key + (i + 1) * 0x9E3779B97F4A7C15ull); }
static inline uint64_t umulhi(uint64_t a, uint64_t b) { return (uint64_t)(((u128)a * b) >> 64); }
static inline int64_t sample_ternary(uint64_t u) { return (int64_t)umulhi(u, 3) - 1; }
static inline uint64_t sample_uniform(uint64_t u, uint64_t q) { return umulhi(u, q); }
static inline int64_t sample_gauss(uint64_t u, const uint64_t *cdt) {
    uint64_t r = u >> 1;
    int mag = 0;
    while (mag < CDT_LEN - 1 && r >= cdt[mag]) mag++;
    return (u & 1) ? -(int64_t)mag : (int64_t)mag;
}
/* CDT for |X| of the discrete Gaussian, sigma = 3.2, thresholds scaled to 2^63 */
void orc_build_cdt(uint64_t *cdt) {
    double z = 1.0;
    for (int k = 1; k < 64; k++) z += 2.0 * exp(-(double)(k * k) / (2.0 * 3.2 * 3.2));
    double cum = 1.0 / z;
    for (int m = 0; m < CDT_LEN; m++) {
        if (m > 0) cum += 2.0 * exp(-(double)(m * m) / (2.0 * 3.2 * 3.2)) / z;
        double t = cum * 9223372036854775808.0;
        cdt[m] = (t >= 9223372036854775808.0) ? 0x8000000000000000ull : (uint64_t)t;
    }
    cdt[CDT_LEN - 1] = 0x8000000000000000ull;
}

/* ------------------------------------------------------------------ */
/* context                                                             */
/* ------------------------------------------------------------------ */
typedef struct {
    uint32_t g;
    uint64_t *key;
} orc_gkey;

typedef struct {
    int log_n, n, slots, L, np;
    uint64_t q[ORC_MAXP];
    uint64_t *psi_br[ORC_MAXP], *psi_br_sh[ORC_MAXP], *ipsi_br[ORC_MAXP], *ipsi_br_sh[ORC_MAXP];
    uint64_t n_inv[ORC_MAXP];
    uint64_t seed;
    double *zr, *zi;  /* zeta^k = exp(i*pi*k/N), k < N */
    int *slot_pos;    /* r_j = (5^j mod 2N - 1)/4 */
    uint64_t cdt[CDT_LEN];
    int8_t *s;
    uint64_t *s_ntt;  /* [np][N] */
    uint64_t *pk;     /* [2][L+1][N] */
    uint64_t *rlk;    /* [L+1][2][np][N] */
    orc_gkey *gk;
    int ngk, capgk;
    int sym_enc;      /* 1 = secret-key encryption, 0 = public key */
} orc_ctx;

static inline uint64_t shoup(uint64_t w, uint64_t q) { return (uint64_t)(((u128)w << 64) / q); }
static inline uint64_t mul_shoup(uint64_t x, uint64_t w, uint64_t wsh, uint64_t q) {
    uint64_t qh = umulhi(x, wsh);
    uint64_t r = x * w - qh * q;
    return r >= q ? r - q : r;
}

/* forward negacyclic NTT, in place, result fully reduced */
void orc_ntt(const orc_ctx *c, int pidx, uint64_t *a) {
    const int n = c->n;
    const uint64_t q = c->q[pidx];
    const uint64_t *w = c->psi_br[pidx], *wsh = c->psi_br_sh[pidx];
    int t = n;
    for (int m = 1; m < n; m <<= 1) {
        t >>= 1;
        for (int i = 0; i < m; i++) {
            const int j1 = 2 * i * t;
            const uint64_t W = w[m + i], Wsh = wsh[m + i];
            for (int j = j1; j < j1 + t; j++) {
                uint64_t u = a[j], v = mul_shoup(a[j + t], W, Wsh, q);
                a[j] = addmod(u, v, q);
                a[j + t] = submod(u, v, q);
            }
        }
    }
}
void orc_intt(const orc_ctx *c, int pidx, uint64_t *a) {
    const int n = c->n;
    const uint64_t q = c->q[pidx];
    const uint64_t *w = c->ipsi_br[pidx], *wsh = c->ipsi_br_sh[pidx];
    int t = 1;
    for (int m = n; m > 1; m >>= 1) {
        int h = m >> 1, j1 = 0;
        for (int i = 0; i < h; i++) {
            const uint64_t W = w[h + i], Wsh = wsh[h + i];
            for (int j = j1; j < j1 + t; j++) {
                uint64_t u = a[j], v = a[j + t];
                a[j] = addmod(u, v, q);
                a[j + t] = mul_shoup(submod(u, v, q), W, Wsh, q);
            }
            j1 += 2 * t;
        }
        t <<= 1;
    }
    const uint64_t ni = c->n_inv[pidx], nish = shoup(ni, q);
    for (int j = 0; j < n; j++) a[j] = mul_shoup(a[j], ni, nish, q);
}

static void gen_gkey(orc_ctx *c, const uint64_t *sprime_ntt, int dom_a, int dom_e, uint64_t id, uint64_t *key);

orc_ctx *orc_create(int log_n, int nq, const uint64_t *primes, uint64_t seed, int sym_enc) {
    if (nq < 1 || nq + 1 > ORC_MAXP || log_n < 2 || log_n > 17) return NULL;
    orc_ctx *c = (orc_ctx *)calloc(1, sizeof(orc_ctx));
    c->log_n = log_n;
    c->n = 1 << log_n;
    c->slots = c->n / 2;
    c->L = nq - 1;
    c->np = nq + 1;
    c->seed = seed;
    c->sym_enc = sym_enc;
    const int n = c->n;
    for (int p = 0; p < c->np; p++) {
        uint64_t q = primes[p];
        c->q[p] = q;
        uint64_t psi = min_psi(q, n), ipsi = invmod(psi, q);
        c->psi_br[p] = malloc(8 * n); c->psi_br_sh[p] = malloc(8 * n);
        c->ipsi_br[p] = malloc(8 * n); c->ipsi_br_sh[p] = malloc(8 * n);
        uint64_t *pw = malloc(8 * n), *ipw = malloc(8 * n);
        pw[0] = 1; ipw[0] = 1;
        for (int i = 1; i < n; i++) { pw[i] = mulmod(pw[i - 1], psi, q); ipw[i] = mulmod(ipw[i - 1], ipsi, q); }
        for (int i = 0; i < n; i++) {
            uint32_t r = bitrev(i, log_n);
            c->psi_br[p][i] = pw[r]; c->psi_br_sh[p][i] = shoup(pw[r], q);
            c->ipsi_br[p][i] = ipw[r]; c->ipsi_br_sh[p][i] = shoup(ipw[r], q);
        }
        free(pw); free(ipw);
        c->n_inv[p] = invmod((uint64_t)n % q, q);
    }
    c->zr = malloc(sizeof(double) * n);
    c->zi = malloc(sizeof(double) * n);
    for (int k = 0; k < n; k++) {
        const double ang = M_PI * (double)k / (double)n;
        c->zr[k] = cos(ang);
        c->zi[k] = sin(ang);
    }
    c->slot_pos = malloc(sizeof(int) * c->slots);
    uint64_t g = 1, two_n = 2ull * n;
    for (int j = 0; j < c->slots; j++) { c->slot_pos[j] = (int)((g - 1) / 4); g = (g * 5) % two_n; }
    orc_build_cdt(c->cdt);

    /* secret key */
    c->s = malloc(n);
    uint64_t ks = orc_stream_key(seed, DOM_SK, 0, 0);
    for (int k = 0; k < n; k++) c->s[k] = (int8_t)sample_ternary(rnd(ks, k));
    c->s_ntt = malloc(8ull * c->np * n);
    for (int p = 0; p < c->np; p++) {
        uint64_t *d = c->s_ntt + (size_t)p * n;
        for (int k = 0; k < n; k++) d[k] = reduce_i64(c->s[k], c->q[p]);
        orc_ntt(c, p, d);
    }
    /* public key over the ciphertext primes */
    const int nl = c->L + 1;
    c->pk = malloc(16ull * nl * n);
    uint64_t *e = malloc(8ull * n);
    uint64_t ke = orc_stream_key(seed, DOM_PK_E, 0, 0);
    for (int i = 0; i < nl; i++) {
        const uint64_t q = c->q[i];
        uint64_t ka = orc_stream_key(seed, DOM_PK_A, 0, i);
        uint64_t *b = c->pk + (size_t)i * n, *a = c->pk + (size_t)(nl + i) * n;
        for (int k = 0; k < n; k++) { a[k] = sample_uniform(rnd(ka, k), q); e[k] = reduce_i64(sample_gauss(rnd(ke, k), c->cdt), q); }
        orc_ntt(c, i, e);
        const uint64_t *s = c->s_ntt + (size_t)i * n;
        for (int k = 0; k < n; k++) b[k] = addmod(submod(0, mulmod(a[k], s[k], q), q), e[k], q);
    }
    free(e);
    return c;
}

void orc_destroy(orc_ctx *c) {
    if (!c) return;
    for (int p = 0; p < c->np; p++) { free(c->psi_br[p]); free(c->psi_br_sh[p]); free(c->ipsi_br[p]); free(c->ipsi_br_sh[p]); }
    free(c->zr); free(c->zi); free(c->slot_pos); free(c->s); free(c->s_ntt); free(c->pk); free(c->rlk);
    for (int i = 0; i < c->ngk; i++) free(c->gk[i].key);
    free(c->gk);
    free(c);
}

int orc_n(const orc_ctx *c) { return c->n; }
void orc_get_tables(const orc_ctx *c, int pidx, uint64_t *psi_br, uint64_t *ipsi_br) {
    memcpy(psi_br, c->psi_br[pidx], 8ull * c->n);
    memcpy(ipsi_br, c->ipsi_br[pidx], 8ull * c->n);
}
void orc_get_cdt(const orc_ctx *c, uint64_t *out) { memcpy(out, c->cdt, sizeof(c->cdt)); }
void orc_get_secret(const orc_ctx *c, int8_t *out) { memcpy(out, c->s, c->n); }
void orc_get_pk(const orc_ctx *c, uint64_t *out) { memcpy(out, c->pk, 16ull * (c->L + 1) * c->n); }

/* key for s' (given in NTT form over all np primes): [L+1 digits][2][np][N] */
static void gen_gkey(orc_ctx *c, const uint64_t *sp, int dom_a, int dom_e, uint64_t id, uint64_t *key) {
    const int n = c->n, np = c->np, P = c->np - 1;
#pragma omp parallel for schedule(static)
    for (int j = 0; j <= c->L; j++) {
        uint64_t *e = malloc(8ull * n);
        uint64_t ke = orc_stream_key(c->seed, dom_e, id, j);
        for (int p = 0; p < np; p++) {
            const uint64_t q = c->q[p];
            uint64_t ka = orc_stream_key(c->seed, dom_a, id, (uint64_t)j * 256 + p);
            uint64_t *b = key + ((size_t)(j * 2 + 0) * np + p) * n;
            uint64_t *a = key + ((size_t)(j * 2 + 1) * np + p) * n;
            for (int k = 0; k < n; k++) { a[k] = sample_uniform(rnd(ka, k), q); e[k] = reduce_i64(sample_gauss(rnd(ke, k), c->cdt), q); }
            orc_ntt(c, p, e);
            const uint64_t *s = c->s_ntt + (size_t)p * n, *s2 = sp + (size_t)p * n;
            const uint64_t pm = c->q[P] % q;
            for (int k = 0; k < n; k++) {
                uint64_t v = addmod(submod(0, mulmod(a[k], s[k], q), q), e[k], q);
                if (p == j) v = addmod(v, mulmod(pm, s2[k], q), q);
                b[k] = v;
            }
        }
        free(e);
    }
}

static const uint64_t *get_rlk(orc_ctx *c) {
    if (!c->rlk) {
        const int n = c->n, np = c->np;
        uint64_t *s2 = malloc(8ull * np * n);
        for (int p = 0; p < np; p++)
            for (int k = 0; k < n; k++) {
                uint64_t v = c->s_ntt[(size_t)p * n + k];
                s2[(size_t)p * n + k] = mulmod(v, v, c->q[p]);
            }
        c->rlk = malloc(8ull * (c->L + 1) * 2 * np * n);
        gen_gkey(c, s2, DOM_RLK_A, DOM_RLK_E, 0, c->rlk);
        free(s2);
    }
    return c->rlk;
}

/* NTT-domain index permutation of X -> X^g */
static void galois_perm(const orc_ctx *c, uint32_t g, uint32_t *perm) {
    const int n = c->n, lg = c->log_n;
    const uint64_t mask = 2ull * n - 1;
    for (int k = 0; k < n; k++) {
        uint64_t e = ((2ull * bitrev(k, lg) + 1) * g) & mask;
        perm[k] = bitrev((uint32_t)((e - 1) >> 1), lg);
    }
}

static const uint64_t *get_gkey(orc_ctx *c, uint32_t g) {
    for (int i = 0; i < c->ngk; i++) if (c->gk[i].g == g) return c->gk[i].key;
    const int n = c->n, np = c->np;
    uint32_t *perm = malloc(4ull * n);
    galois_perm(c, g, perm);
    uint64_t *sg = malloc(8ull * np * n);
    for (int p = 0; p < np; p++)
        for (int k = 0; k < n; k++) sg[(size_t)p * n + k] = c->s_ntt[(size_t)p * n + perm[k]];
    free(perm);
    uint64_t *key = malloc(8ull * (c->L + 1) * 2 * np * n);
    gen_gkey(c, sg, DOM_GAL_A, DOM_GAL_E, g, key);
    free(sg);
    if (c->ngk == c->capgk) { c->capgk = c->capgk ? 2 * c->capgk : 8; c->gk = realloc(c->gk, sizeof(orc_gkey) * c->capgk); }
    c->gk[c->ngk].g = g;
    c->gk[c->ngk].key = key;
    c->ngk++;
    return key;
}
void orc_get_relin_key(orc_ctx *c, uint64_t *out) { memcpy(out, get_rlk(c), 8ull * (c->L + 1) * 2 * c->np * c->n); }
void orc_get_galois_key(orc_ctx *c, uint32_t g, uint64_t *out) { memcpy(out, get_gkey(c, g), 8ull * (c->L + 1) * 2 * c->np * c->n); }

/* ------------------------------------------------------------------ */
/* encode / decode (canonical embedding, slot j <-> zeta^(5^j))         */
/* ------------------------------------------------------------------ */
static void fft_core(const orc_ctx *c, double *re, double *im, int inverse) {
    const int S = c->slots;
    int lg = 0;
    while ((1 << lg) < S) lg++;
    for (int i = 0; i < S; i++) {
        int j = (int)bitrev(i, lg);
        if (j > i) { double t = re[i]; re[i] = re[j]; re[j] = t; t = im[i]; im[i] = im[j]; im[j] = t; }
    }
    for (int len = 2; len <= S; len <<= 1) {
        const int half = len >> 1, step = S / len;
        for (int i = 0; i < S; i += len)
            for (int j = 0; j < half; j++) {
                const int idx = 4 * j * step;
                const double wr = c->zr[idx], wi = inverse ? -c->zi[idx] : c->zi[idx];
                const double ar = re[i + j], ai = im[i + j];
                const double br = re[i + j + half], bi = im[i + j + half];
                const double tr = br * wr - bi * wi;
                const double ti = br * wi + bi * wr;
                re[i + j] = ar + tr; im[i + j] = ai + ti;
                re[i + j + half] = ar - tr; im[i + j + half] = ai - ti;
            }
    }
}

/* values (nvals <= S reals) -> integer coefficients m[N] at the given scale */
void orc_encode_coeffs(const orc_ctx *c, const double *vals, int nvals, double scale, int64_t *m) {
    const int S = c->slots;
    double *re = calloc(S, sizeof(double)), *im = calloc(S, sizeof(double));
    for (int j = 0; j < nvals; j++) re[c->slot_pos[j]] = vals[j];
    fft_core(c, re, im, 1);
    const double f = scale / (double)S;
    for (int k = 0; k < S; k++) {
        const double yr = re[k], yi = im[k];
        const double xr = yr * c->zr[k] + yi * c->zi[k];
        const double xi = yi * c->zr[k] - yr * c->zi[k];
        m[k] = llrint(xr * f);
        m[k + S] = llrint(xi * f);
    }
    free(re); free(im);
}

/* centered integer coefficients -> slot values (real and imaginary parts) */
void orc_decode_coeffs(const orc_ctx *c, const int64_t *m, double scale, double *out_re, double *out_im) {
    const int S = c->slots;
    double *re = malloc(sizeof(double) * S), *im = malloc(sizeof(double) * S);
    for (int k = 0; k < S; k++) {
        const double ur = (double)m[k] / scale, ui = (double)m[k + S] / scale;
        re[k] = ur * c->zr[k] - ui * c->zi[k];
        im[k] = ur * c->zi[k] + ui * c->zr[k];
    }
    fft_core(c, re, im, 0);
    for (int j = 0; j < S; j++) {
        out_re[j] = re[c->slot_pos[j]];
        if (out_im) out_im[j] = im[c->slot_pos[j]];
    }
    free(re); free(im);
}

/* plaintext in NTT form at level l: [l+1][N] */
void orc_encode(const orc_ctx *c, const double *vals, int nvals, int level, double scale, uint64_t *pt) {
    const int n = c->n;
    int64_t *m = malloc(8ull * n);
    orc_encode_coeffs(c, vals, nvals, scale, m);
    for (int i = 0; i <= level; i++) {
        uint64_t *d = pt + (size_t)i * n;
        for (int k = 0; k < n; k++) d[k] = reduce_i64(m[k], c->q[i]);
        orc_ntt(c, i, d);
    }
    free(m);
}

/* fresh encryption at level l with nonce -> [2][l+1][N] */
void orc_encrypt(const orc_ctx *c, const double *vals, int nvals, int level, double scale, uint64_t nonce, uint64_t *ct) {
    const int n = c->n, nl = level + 1;
    int64_t *m = malloc(8ull * n);
    orc_encode_coeffs(c, vals, nvals, scale, m);
    uint64_t kv = orc_stream_key(c->seed, DOM_ENC_V, nonce, 0);
    uint64_t ke0 = orc_stream_key(c->seed, DOM_ENC_E0, nonce, 0);
    uint64_t ke1 = orc_stream_key(c->seed, DOM_ENC_E1, nonce, 0);
    int64_t *v = malloc(8ull * n), *e0 = malloc(8ull * n), *e1 = malloc(8ull * n);
    for (int k = 0; k < n; k++) {
        v[k] = sample_ternary(rnd(kv, k));
        e0[k] = sample_gauss(rnd(ke0, k), c->cdt) + m[k];
        e1[k] = sample_gauss(rnd(ke1, k), c->cdt);
    }
    const int Ltop = c->L;
#pragma omp parallel for schedule(static)
    for (int i = 0; i < nl; i++) {
        const uint64_t q = c->q[i];
        uint64_t *c0 = ct + (size_t)i * n, *c1 = ct + (size_t)(nl + i) * n;
        if (c->sym_enc) {
            uint64_t ka = orc_stream_key(c->seed, DOM_ENC_A, nonce, i);
            for (int k = 0; k < n; k++) { c1[k] = sample_uniform(rnd(ka, k), q); c0[k] = reduce_i64(e0[k], q); }
            orc_ntt(c, i, c0);
            const uint64_t *s = c->s_ntt + (size_t)i * n;
            for (int k = 0; k < n; k++) c0[k] = submod(c0[k], mulmod(c1[k], s[k], q), q);
        } else {
            uint64_t *vv = malloc(8ull * n);
            for (int k = 0; k < n; k++) { vv[k] = reduce_i64(v[k], q); c0[k] = reduce_i64(e0[k], q); c1[k] = reduce_i64(e1[k], q); }
            orc_ntt(c, i, vv); orc_ntt(c, i, c0); orc_ntt(c, i, c1);
            const uint64_t *p0 = c->pk + (size_t)i * n, *p1 = c->pk + (size_t)(Ltop + 1 + i) * n;
            for (int k = 0; k < n; k++) {
                c0[k] = addmod(mulmod(vv[k], p0[k], q), c0[k], q);
                c1[k] = addmod(mulmod(vv[k], p1[k], q), c1[k], q);
            }
            free(vv);
        }
    }
    free(m); free(v); free(e0); free(e1);
}

/* decrypt (deg 1 or 2) on limb q0 and decode; ct = [deg+1][l+1][N] */
void orc_decrypt_coeffs(const orc_ctx *c, const uint64_t *ct, int deg, int level, int64_t *m) {
    const int n = c->n, nl = level + 1;
    const uint64_t q = c->q[0];
    uint64_t *x = malloc(8ull * n);
    const uint64_t *s = c->s_ntt;
    for (int k = 0; k < n; k++) {
        uint64_t v = addmod(ct[k], mulmod(ct[(size_t)nl * n + k], s[k], q), q);
        if (deg == 2) v = addmod(v, mulmod(ct[(size_t)2 * nl * n + k], mulmod(s[k], s[k], q), q), q);
        x[k] = v;
    }
    orc_intt(c, 0, x);
    for (int k = 0; k < n; k++) m[k] = x[k] > (q >> 1) ? -(int64_t)(q - x[k]) : (int64_t)x[k];
    free(x);
}
void orc_decrypt_decode(const orc_ctx *c, const uint64_t *ct, int deg, int level, double scale, double *out_re) {
    int64_t *m = malloc(8ull * c->n);
    orc_decrypt_coeffs(c, ct, deg, level, m);
    orc_decode_coeffs(c, m, scale, out_re, NULL);
    free(m);
}

/* ------------------------------------------------------------------ */
/* ring operations                                                     */
/* ------------------------------------------------------------------ */
void orc_add(const orc_ctx *c, const uint64_t *a, const uint64_t *b, int deg, int level, uint64_t *out) {
    const int n = c->n, nl = level + 1;
    for (int p = 0; p <= deg; p++)
        for (int i = 0; i < nl; i++) {
            const uint64_t q = c->q[i];
            size_t o = ((size_t)p * nl + i) * n;
            for (int k = 0; k < n; k++) out[o + k] = addmod(a[o + k], b[o + k], q);
        }
}
void orc_sub(const orc_ctx *c, const uint64_t *a, const uint64_t *b, int deg, int level, uint64_t *out) {
    const int n = c->n, nl = level + 1;
    for (int p = 0; p <= deg; p++)
        for (int i = 0; i < nl; i++) {
            const uint64_t q = c->q[i];
            size_t o = ((size_t)p * nl + i) * n;
            for (int k = 0; k < n; k++) out[o + k] = submod(a[o + k], b[o + k], q);
        }
}
/* (a0,a1) x (b0,b1) -> (a0b0, a0b1+a1b0, a1b1) */
void orc_tensor(const orc_ctx *c, const uint64_t *a, const uint64_t *b, int level, uint64_t *d) {
    const int n = c->n, nl = level + 1;
    for (int i = 0; i < nl; i++) {
        const uint64_t q = c->q[i];
        const size_t o0 = (size_t)i * n, o1 = (size_t)(nl + i) * n, o2 = (size_t)(2 * nl + i) * n;
        for (int k = 0; k < n; k++) {
            uint64_t a0 = a[o0 + k], a1 = a[o1 + k], b0 = b[o0 + k], b1 = b[o1 + k];
            d[o0 + k] = mulmod(a0, b0, q);
            d[o1 + k] = addmod(mulmod(a0, b1, q), mulmod(a1, b0, q), q);
            d[o2 + k] = mulmod(a1, b1, q);
        }
    }
}
void orc_mul_plain(const orc_ctx *c, const uint64_t *ct, const uint64_t *pt, int deg, int level, uint64_t *out) {
    const int n = c->n, nl = level + 1;
    for (int p = 0; p <= deg; p++)
        for (int i = 0; i < nl; i++) {
            const uint64_t q = c->q[i];
            size_t o = ((size_t)p * nl + i) * n;
            for (int k = 0; k < n; k++) out[o + k] = mulmod(ct[o + k], pt[(size_t)i * n + k], q);
        }
}
void orc_mul_scalar(const orc_ctx *c, const uint64_t *ct, int64_t s, int deg, int level, uint64_t *out) {
    const int n = c->n, nl = level + 1;
    for (int p = 0; p <= deg; p++)
        for (int i = 0; i < nl; i++) {
            const uint64_t q = c->q[i], sv = reduce_i64(s, q);
            size_t o = ((size_t)p * nl + i) * n;
            for (int k = 0; k < n; k++) out[o + k] = mulmod(ct[o + k], sv, q);
        }
}
/* add the constant polynomial s (all NTT values = s) to poly 0 */
void orc_add_const(const orc_ctx *c, uint64_t *ct, int64_t s, int level) {
    const int n = c->n;
    for (int i = 0; i <= level; i++) {
        const uint64_t q = c->q[i], sv = reduce_i64(s, q);
        for (int k = 0; k < n; k++) ct[(size_t)i * n + k] = addmod(ct[(size_t)i * n + k], sv, q);
    }
}
/* keep limbs 0..to of each poly */
void orc_drop_level(const orc_ctx *c, const uint64_t *ct, int deg, int from, int to, uint64_t *out) {
    const int n = c->n;
    for (int p = 0; p <= deg; p++)
        memcpy(out + (size_t)p * (to + 1) * n, ct + (size_t)p * (from + 1) * n, 8ull * (to + 1) * n);
}

/* rescale: divide by q_l with rounding, level l -> l-1 */
void orc_rescale(const orc_ctx *c, const uint64_t *ct, int deg, int level, uint64_t *out) {
    const int n = c->n, nl = level + 1;
    const uint64_t ql = c->q[level];
    uint64_t *y = malloc(8ull * n), *z = malloc(8ull * n);
    for (int p = 0; p <= deg; p++) {
        memcpy(y, ct + ((size_t)p * nl + level) * n, 8ull * n);
        orc_intt(c, level, y);
        for (int i = 0; i < level; i++) {
            const uint64_t q = c->q[i], inv = invmod(ql % q, q);
            for (int k = 0; k < n; k++) z[k] = lift_centered(y[k], ql, q);
            orc_ntt(c, i, z);
            const uint64_t *src = ct + ((size_t)p * nl + i) * n;
            uint64_t *dst = out + ((size_t)p * level + i) * n;
            for (int k = 0; k < n; k++) dst[k] = mulmod(submod(src[k], z[k], q), inv, q);
        }
    }
    free(y); free(z);
}

/* hybrid key switch, dnum = l+1 single-prime digits, one special prime P.
 * cpoly: [l+1][N] NTT; key: [L+1][2][np][N]; out: [2][l+1][N] */
/* inner product accumulators acc[2][l+2][N] (targets q0..ql, P) of the hybrid key switch */
static void keyswitch_acc(orc_ctx *c, const uint64_t *cpoly, int level, const uint64_t *key, uint64_t *acc) {
    const int n = c->n, nl = level + 1, np = c->np, P = np - 1;
    const int nt = nl + 1; /* target primes q0..ql, P */
    memset(acc, 0, 16ull * nt * n);
    /* the digits' coefficient forms first, then one independent work item per target prime
       (threads never share an accumulator; per-target accumulation order is j = 0..l) */
    uint64_t *xs = malloc(8ull * nl * n);
#pragma omp parallel for schedule(static)
    for (int j = 0; j < nl; j++) {
        memcpy(xs + (size_t)j * n, cpoly + (size_t)j * n, 8ull * n);
        orc_intt(c, j, xs + (size_t)j * n);
    }
#pragma omp parallel for schedule(dynamic)
    for (int t = 0; t < nt; t++) {
        uint64_t *d = malloc(8ull * n);
        const int pidx = t < nl ? t : P;
        const uint64_t q = c->q[pidx];
        for (int j = 0; j < nl; j++) {
            const uint64_t *x = xs + (size_t)j * n;
            if (t == j) memcpy(d, cpoly + (size_t)j * n, 8ull * n);
            else {
                for (int k = 0; k < n; k++) d[k] = lift_centered(x[k], c->q[j], q);
                orc_ntt(c, pidx, d);
            }
            for (int b = 0; b < 2; b++) {
                const uint64_t *kk = key + ((size_t)(j * 2 + b) * np + pidx) * n;
                uint64_t *a = acc + ((size_t)b * nt + t) * n;
                for (int k = 0; k < n; k++) a[k] = addmod(a[k], mulmod(d[k], kk[k], q), q);
            }
        }
        free(d);
    }
    free(xs);
}

/* hybrid key switch, dnum = l+1 single-prime digits, one special prime P.
 * cpoly: [l+1][N] NTT; key: [L+1][2][np][N]; out: [2][l+1][N] */
void orc_keyswitch(const orc_ctx *c, const uint64_t *cpoly, int level, const uint64_t *key, uint64_t *out) {
    const int n = c->n, nl = level + 1, np = c->np, P = np - 1;
    const int nt = nl + 1;
    uint64_t *acc = malloc(16ull * nt * n);
    keyswitch_acc((orc_ctx *)c, cpoly, level, key, acc);
    uint64_t *x = malloc(8ull * n), *d = malloc(8ull * n);
    const uint64_t Pq = c->q[P];
    for (int b = 0; b < 2; b++) {
        memcpy(x, acc + ((size_t)b * nt + nl) * n, 8ull * n);
        orc_intt(c, P, x);
        for (int i = 0; i < nl; i++) {
            const uint64_t q = c->q[i], pinv = invmod(Pq % q, q);
            for (int k = 0; k < n; k++) d[k] = lift_centered(x[k], Pq, q);
            orc_ntt(c, i, d);
            const uint64_t *a = acc + ((size_t)b * nt + i) * n;
            uint64_t *o = out + ((size_t)b * nl + i) * n;
            for (int k = 0; k < n; k++) o[k] = mulmod(submod(a[k], d[k], q), pinv, q);
        }
    }
    free(acc); free(x); free(d);
}

/* degree-2 -> degree-1 */
void orc_relin(orc_ctx *c, const uint64_t *d3, int level, uint64_t *out) {
    const int n = c->n, nl = level + 1;
    uint64_t *ks = malloc(16ull * nl * n);
    orc_keyswitch(c, d3 + (size_t)2 * nl * n, level, get_rlk(c), ks);
    for (int b = 0; b < 2; b++)
        for (int i = 0; i < nl; i++) {
            const uint64_t q = c->q[i];
            size_t o = ((size_t)b * nl + i) * n;
            for (int k = 0; k < n; k++) out[o + k] = addmod(d3[o + k], ks[o + k], q);
        }
    free(ks);
}

/* Fused relinearisation + rescale: with acc = ModUp/inner(d2)
 * over {q_0..q_l, P}, X = P*d_{0,1} + acc_{0,1} is divided by P*q_l with rounding:
 *   out_i = (X_i - lift([X]_{P q_l})) * (P q_l)^-1 mod q_i,   i < l
 * where [X]_{P q_l} is the centred CRT combination of X mod P and X mod q_l.
 * d3: [3][l+1][N] -> out [2][l][N] */
static void keyswitch_acc(orc_ctx *c, const uint64_t *cpoly, int level, const uint64_t *key, uint64_t *acc);
void orc_relin_rescale(orc_ctx *c, const uint64_t *d3, int level, uint64_t *out) {
    const int n = c->n, nl = level + 1, nt = nl + 1, np = c->np, P = np - 1;
    const uint64_t Pq = c->q[P], ql = c->q[level];
    uint64_t *acc = malloc(16ull * nt * n);
    keyswitch_acc(c, d3 + (size_t)2 * nl * n, level, get_rlk(c), acc);
    uint64_t *yqs = malloc(16ull * n), *yps = malloc(16ull * n);
    const uint64_t pinv_ql = invmod(Pq % ql, ql), p_ql = Pq % ql;
#pragma omp parallel for schedule(static)
    for (int b = 0; b < 2; b++) {
        const uint64_t *ab = acc + (size_t)b * nt * n, *db = d3 + (size_t)b * nl * n;
        uint64_t *yq = yqs + (size_t)b * n, *yp = yps + (size_t)b * n;
        for (int k = 0; k < n; k++) {
            yq[k] = addmod(mulmod(p_ql, db[(size_t)level * n + k], ql), ab[(size_t)level * n + k], ql);
            yp[k] = ab[(size_t)nl * n + k];
        }
        orc_intt(c, level, yq);
        orc_intt(c, P, yp);
    }
#pragma omp parallel for schedule(dynamic) collapse(2)
    for (int b = 0; b < 2; b++) {
        for (int i = 0; i < level; i++) {
            const uint64_t *ab = acc + (size_t)b * nt * n, *db = d3 + (size_t)b * nl * n;
            const uint64_t *yq = yqs + (size_t)b * n, *yp = yps + (size_t)b * n;
            uint64_t *z = malloc(8ull * n);
            const uint64_t q = c->q[i], pm = Pq % q, pqm = mulmod(pm, ql % q, q);
            const uint64_t inv = invmod(pqm, q);
            for (int k = 0; k < n; k++) {
                /* x = yp + P * t, t = (yq - yp) * P^-1 mod ql, x in [0, P ql) */
                const uint64_t t = mulmod(submod(yq[k], yp[k] % ql, ql), pinv_ql, ql);
                uint64_t v = addmod(yp[k] % q, mulmod(pm, t % q, q), q);
                const int neg = (t > (ql - 1) / 2) || (t == (ql - 1) / 2 && yp[k] > Pq / 2);
                if (neg) v = submod(v, pqm, q);
                z[k] = v;
            }
            orc_ntt(c, i, z);
            uint64_t *o = out + ((size_t)b * level + i) * n;
            for (int k = 0; k < n; k++) {
                const uint64_t x = addmod(mulmod(pm, db[(size_t)i * n + k], q), ab[(size_t)i * n + k], q);
                o[k] = mulmod(submod(x, z[k], q), inv, q);
            }
            free(z);
        }
    }
    free(acc); free(yqs); free(yps);
}

uint32_t orc_galois_elt(const orc_ctx *c, int64_t steps) {
    int64_t S = c->slots;
    int64_t r = ((steps % S) + S) % S;
    uint64_t g = 1, two_n = 2ull * c->n;
    for (int64_t i = 0; i < r; i++) g = (g * 5) % two_n;
    return (uint32_t)g;
}

/* cyclic LEFT rotation by `steps` slots (engine.py:232-236) */
void orc_rotate(orc_ctx *c, const uint64_t *ct, int level, int64_t steps, uint64_t *out) {
    const int n = c->n, nl = level + 1;
    uint32_t g = orc_galois_elt(c, steps);
    if (g == 1) { memcpy(out, ct, 16ull * nl * n); return; }
    const uint64_t *key = get_gkey(c, g);
    uint32_t *perm = malloc(4ull * n);
    galois_perm(c, g, perm);
    uint64_t *r = malloc(16ull * nl * n), *ks = malloc(16ull * nl * n);
    for (int p = 0; p < 2; p++)
        for (int i = 0; i < nl; i++) {
            const uint64_t *src = ct + ((size_t)p * nl + i) * n;
            uint64_t *dst = r + ((size_t)p * nl + i) * n;
            for (int k = 0; k < n; k++) dst[k] = src[perm[k]];
        }
    orc_keyswitch(c, r + (size_t)nl * n, level, key, ks);
    for (int i = 0; i < nl; i++) {
        const uint64_t q = c->q[i];
        for (int k = 0; k < n; k++) {
            out[(size_t)i * n + k] = addmod(r[(size_t)i * n + k], ks[(size_t)i * n + k], q);
            out[(size_t)(nl + i) * n + k] = ks[(size_t)(nl + i) * n + k];
        }
    }
    free(perm); free(r); free(ks);
}

/* mul = tensor -> relin -> rescale (level l -> l-1) */
void orc_mul(orc_ctx *c, const uint64_t *a, const uint64_t *b, int level, uint64_t *out) {
    const int n = c->n, nl = level + 1;
    uint64_t *d = malloc(24ull * nl * n);
    orc_tensor(c, a, b, level, d);
    orc_relin_rescale(c, d, level, out);
    free(d);
}

/* ------------------------------------------------------------------ */
/* fused drivers                                                       */
/* ------------------------------------------------------------------ */

/* matmul_outer (multicipher.py:88-103), fused: sum_k tensor(L_k, R_k) mod q,
 * then one relinearisation and one rescale.  Ls/Rs: n pointers to [2][l+1][N];
 * out: [2][l][N]. */
void orc_matmul_outer(orc_ctx *c, const uint64_t *const *Ls, const uint64_t *const *Rs, int count, int level, uint64_t *out) {
    const int n = c->n, nl = level + 1;
    uint64_t *d = calloc((size_t)3 * nl * n, 8);
    /* (limb, coefficient chunk) work items so every host thread has work (the per-coefficient
       accumulation order over t is unchanged) */
    const int nch = n >= 64 ? 32 : 1;
#pragma omp parallel for schedule(static) collapse(2)
    for (int i = 0; i < nl; i++) {
        for (int ch = 0; ch < nch; ch++) {
        const uint64_t q = c->q[i];
        const size_t o0 = (size_t)i * n, o1 = (size_t)(nl + i) * n, o2 = (size_t)(2 * nl + i) * n;
        const int k0 = ch * (n / nch), k1 = k0 + n / nch;
        for (int t = 0; t < count; t++) {
            const uint64_t *a = Ls[t], *b = Rs[t];
            for (int k = k0; k < k1; k++) {
                uint64_t a0 = a[o0 + k], a1 = a[o1 + k], b0 = b[o0 + k], b1 = b[o1 + k];
                d[o0 + k] = addmod(d[o0 + k], mulmod(a0, b0, q), q);
                d[o1 + k] = addmod(d[o1 + k], addmod(mulmod(a0, b1, q), mulmod(a1, b0, q), q), q);
                d[o2 + k] = addmod(d[o2 + k], mulmod(a1, b1, q), q);
            }
        }
        }
    }
    orc_relin_rescale(c, d, level, out);
    free(d);
}

/* Column-domain convolution (multicipher.py:123-162), generalised to C input
 * channels and F filters (the paper's channel sum):
 *   Y[f][o] = rescale( mask * ( sum_{c,p,q} w[f][c][p][q] * rot(X[c][out_cols[o]+q], p)
 *                               + bias[f] ) )
 * w: int64 [F][C][k][k] (already quantised), bias_res: [F][l+1] residues of
 * the bias integer at the accumulator scale (it can exceed 64 bits),
 * mask: plaintext [l+1][N] NTT.  X: C*W pointers,
 * Y: F*nout pointers, each [2][l][N]. */
void orc_conv_columns(orc_ctx *c, const uint64_t *const *X, int C, int W, int k, const int64_t *w,
                      const uint64_t *bias_res, int F, const int *out_cols, int nout, const uint64_t *mask,
                      int level, uint64_t *const *Y) {
    const int n = c->n, nl = level + 1;
    const size_t ctw = (size_t)2 * nl * n;
    /* rotated copies R[c][j][p] for p >= 1 where some nonzero tap needs them */
    uint64_t **R = calloc((size_t)C * W * k, sizeof(uint64_t *));
    for (int ch = 0; ch < C; ch++)
        for (int j = 0; j < W; j++)
            for (int p = 1; p < k; p++) {
                int need = 0;
                for (int f = 0; f < F && !need; f++)
                    for (int qq = 0; qq < k && !need; qq++) {
                        if (w[((f * C + ch) * k + p) * k + qq] == 0) continue;
                        for (int o = 0; o < nout; o++) if (out_cols[o] + qq == j) { need = 1; break; }
                    }
                if (!need) continue;
                uint64_t *dst = malloc(8 * ctw);
                orc_rotate(c, X[ch * W + j], level, p, dst);
                R[((size_t)ch * W + j) * k + p] = dst;
            }
#pragma omp parallel for schedule(dynamic) collapse(2)
    for (int f = 0; f < F; f++)
        for (int o = 0; o < nout; o++) {
            uint64_t *acc = calloc(ctw, 8);
            for (int ch = 0; ch < C; ch++)
                for (int qq = 0; qq < k; qq++)
                    for (int p = 0; p < k; p++) {
                        const int64_t wt = w[((f * C + ch) * k + p) * k + qq];
                        if (wt == 0) continue;
                        const int j = out_cols[o] + qq;
                        const uint64_t *src = p == 0 ? X[ch * W + j] : R[((size_t)ch * W + j) * k + p];
                        for (int pp = 0; pp < 2; pp++)
                            for (int i = 0; i < nl; i++) {
                                const uint64_t q = c->q[i], wv = reduce_i64(wt, q);
                                const size_t off = ((size_t)pp * nl + i) * n;
                                for (int kk = 0; kk < n; kk++) acc[off + kk] = addmod(acc[off + kk], mulmod(src[off + kk], wv, q), q);
                            }
                    }
            for (int i = 0; i < nl; i++) {
                const uint64_t q = c->q[i], bv = bias_res[(size_t)f * nl + i] % q;
                for (int kk = 0; kk < n; kk++) acc[(size_t)i * n + kk] = addmod(acc[(size_t)i * n + kk], bv, q);
            }
            orc_mul_plain(c, acc, mask, 1, level, acc);
            orc_rescale(c, acc, 1, level, Y[f * nout + o]);
            free(acc);
        }
    for (size_t i = 0; i < (size_t)C * W * k; i++) free(R[i]);
    free(R);
}

/* poly_activation (pipeline.py:180-197) fused, see DESIGN.md section 4.3.
 * x at level l (scale s_l), x' = x with limbs 0..l-1 (same scale):
 *   x2  = rescale(relin(x (x) x))                                   level l-1, s_{l-1}
 *   c3 == 0:  pre = x2 * kc[1] + x' * kc[2]                         level l-1, s_{l-1}^2
 *   c3 != 0:  inner = rescale(x * kc[0]) + kc[1]                    level l-1, s_{l-1}
 *             pre = relin(x2 (x) inner) + x' * kc[2]                level l-1, s_{l-1}^2
 *   out = rescale(pre) + kc[3]                                      level l-2, s_{l-2}
 * kc = {round(c3 s_l), round(c2 s_{l-1}), round(c1 s_{l-1}^2 / s_l), round(c0 s_{l-2})}.
 * x: [2][l+1][N] -> out [2][l-1][N] */
void orc_poly_activation(orc_ctx *c, const uint64_t *x, int level, const int64_t *kc, int c3_zero, uint64_t *out) {
    const int n = c->n, nl = level + 1;
    const size_t w1 = (size_t)2 * level * n;
    uint64_t *x2 = malloc(8 * w1), *xd = malloc(8 * w1), *tmp = malloc(8 * 2 * nl * n);
    orc_mul(c, x, x, level, x2);
    orc_drop_level(c, x, 1, level, level - 1, xd);
    orc_mul_scalar(c, xd, kc[2], 1, level - 1, xd);
    if (c3_zero) {
        uint64_t *pre = malloc(8 * w1);
        orc_mul_scalar(c, x2, kc[1], 1, level - 1, pre);
        orc_add(c, pre, xd, 1, level - 1, pre);
        orc_rescale(c, pre, 1, level - 1, out);
        free(pre);
    } else {
        uint64_t *inner = malloc(8 * w1), *d3 = malloc(8 * 3 * (size_t)level * n);
        orc_mul_scalar(c, x, kc[0], 1, level, tmp);
        orc_rescale(c, tmp, 1, level, inner);
        orc_add_const(c, inner, kc[1], level - 1);
        orc_tensor(c, x2, inner, level - 1, d3);
        orc_add(c, d3, xd, 1, level - 1, d3); /* x' k1 joins (d0, d1) before the fused relin+rescale */
        orc_relin_rescale(c, d3, level - 1, out);
        free(inner); free(d3);
    }
    orc_add_const(c, out, kc[3], level - 2);
    free(x2); free(xd); free(tmp);
}

/* single-limb helpers for unit tests */
void orc_ntt_limb(const orc_ctx *c, int pidx, uint64_t *a) { orc_ntt(c, pidx, a); }
void orc_intt_limb(const orc_ctx *c, int pidx, uint64_t *a) { orc_intt(c, pidx, a); }
void orc_galois_perm(const orc_ctx *c, uint32_t g, uint32_t *perm) { galois_perm(c, g, perm); }
