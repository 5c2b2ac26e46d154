// abi.cu -- extern "C" entry points of libvrhe.so (declared in include/vrhe.h)
// and context construction (prime tables, NTT twiddles, FFT tables, keys).
#include <math.h>

#include <cstring>
#include <map>
#include <mutex>

#include "../../include/vrhe.h"
#include "encode.cuh"
#include "graph.cuh"

struct vr_ctx {
    vr::Ctx c;
};

// A ciphertext owned through the C-ABI (engine.py:140-150 Ciphertext): device residues
// [degree+1][level+1][N] in NTT form plus the level / scale bookkeeping the engine keeps.
struct vr_ct {
    uint64_t *data = nullptr;
    int level = 0, degree = 1;
    double scale = 1.0;
};

namespace {

thread_local std::string g_err;

typedef unsigned __int128 u128h;

uint64_t h_mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128h)a * b) % q); }
uint64_t h_pow(uint64_t b, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = h_mulmod(r, b, q);
        b = h_mulmod(b, b, q);
        e >>= 1;
    }
    return r;
}
uint64_t h_inv(uint64_t a, uint64_t q) { return h_pow(a % q, q - 2, q); }
uint64_t h_shoup(uint64_t w, uint64_t q) { return (uint64_t)(((u128h)w << 64) / q); }
uint32_t h_brev(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

// minimal primitive 2N-th root of unity (same rule as the oracle)
uint64_t h_min_psi(uint64_t q, int n) {
    const uint64_t two_n = 2ull * n;
    uint64_t psi = 0;
    for (uint64_t g = 2;; g++) {
        uint64_t x = h_pow(g, (q - 1) / two_n, q);
        if (h_pow(x, n, q) == q - 1) { psi = x; break; }
    }
    uint64_t best = psi, sq = h_mulmod(psi, psi, q), cur = psi;
    for (int k = 1; k < n; k++) {
        cur = h_mulmod(cur, sq, q);
        if (cur < best) best = cur;
    }
    return best;
}

void build_cdt(uint64_t *cdt) {
    double z = 1.0;
    for (int k = 1; k < 64; k++) z += 2.0 * exp(-(double)(k * k) / (2.0 * 3.2 * 3.2));
    double cum = 1.0 / z;
    for (int m = 0; m < vr::CDT_LEN; m++) {
        if (m > 0) cum += 2.0 * exp(-(double)(m * m) / (2.0 * 3.2 * 3.2)) / z;
        double t = cum * 9223372036854775808.0;
        cdt[m] = (t >= 9223372036854775808.0) ? 0x8000000000000000ull : (uint64_t)t;
    }
    cdt[vr::CDT_LEN - 1] = 0x8000000000000000ull;
}

template <class T>
T *upload(vr::Ctx &c, const std::vector<T> &h) {
    T *d = nullptr;
    VR_CUDA(cudaMalloc((void **)&d, sizeof(T) * h.size()));
    VR_CUDA(cudaMemcpy(d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
    return d;
}

template <class F>
int guard(F &&f) {
    try {
        f();
        return VR_OK;
    } catch (const vr::VrError &e) {
        g_err = e.what();
        return e.code;
    } catch (const std::exception &e) {
        g_err = e.what();
        return VR_ERR_ENGINE;
    }
}

std::vector<const uint64_t *> vec(const uint64_t *const *p, size_t n) { return std::vector<const uint64_t *>(p, p + n); }
std::vector<const uint64_t *> vecm(uint64_t *const *p, size_t n) { return std::vector<const uint64_t *>(p, p + n); }

void check_level(const vr::Ctx &c, int level) {
    if (level < 0 || level > c.L) throw vr::VrError(VR_ERR_ENGINE, "level out of range");
}

// Release everything a (possibly partially constructed) context owns.  Errors are ignored:
// this runs on the vr_ctx_create failure path and from vr_ctx_destroy.
void destroy_ctx(vr_ctx *h) {
    vr::Ctx &c = h->c;
    cudaSetDevice(c.device);
    for (cudaStream_t s : {c.own, c.aux, c.hi, c.stream, c.side})
        if (s) cudaStreamSynchronize(s);
    for (cudaStream_t s : c.slot_stream)
        if (s) cudaStreamSynchronize(s);
    vr::graphs_release(c);
    try {
        vr::comm_destroy(c);
    } catch (...) {
    }
    void *ptrs[] = {c.tw2, c.itw2, c.twd, c.itwd, c.liftk, c.kshift, c.ntt_const, c.inv_tab, c.rr_tab, c.zr, c.zi, c.ftw,
                    c.slot_pos, c.pos_slot, c.cdt, c.rlk, c.s_ntt, c.s_sh, c.pk, c.arena};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    for (auto &kv : c.gkeys) cudaFree(kv.second);
    for (auto &e : c.tables)
        if (e.dev) cudaFree(e.dev);
    for (auto &tk : c.tickets) {
        if (tk.host) cudaFreeHost(tk.host);
        if (tk.done) cudaEventDestroy(tk.done);
    }
    c.tickets.clear();
    for (auto &b : c.big_free) cudaFree(b.second);
    for (auto &kv : c.parked) {
        if (kv.second.arena) cudaFree(kv.second.arena);
        for (auto &b : kv.second.big_free) cudaFree(b.second);
    }
    for (cudaEvent_t e : {c.ev_fork, c.ev_join, c.ev_hi, c.ev_hi_done})
        if (e) cudaEventDestroy(e);
    for (int i = 0; i < vr::Ctx::kStageSlots; i++)
        if (c.stage_evt[i]) cudaEventDestroy(c.stage_evt[i]);
    if (c.stage) cudaFreeHost(c.stage);
    // the private streams only; a user stream installed by vr_set_stream belongs to the caller
    // (the slot streams are process-wide, graph.cu, and stay)
    for (cudaStream_t s : {c.own, c.aux, c.hi, c.side})
        if (s) cudaStreamDestroy(s);
    cudaGetLastError();
    delete h;
}

}  // namespace

namespace vr {
unsigned long long g_launches = 0;

void ensure_smem(Ctx &c, const void *kern, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, size_t> done;
    std::lock_guard<std::mutex> lock(mu);
    size_t &have = done[{c.device, kern}];
    if (smem <= have) return;
    int cur = c.device;
    VR_CUDA(cudaGetDevice(&cur));
    if (cur != c.device) VR_CUDA(cudaSetDevice(c.device));
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cur != c.device) cudaSetDevice(cur);
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw VrError(4, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    }
    have = smem;
}

const void *const *cached_table(Ctx &c, const void *const *ptrs, size_t n) {
    static const void *empty_slot = nullptr;
    if (n == 0) n = 1, ptrs = &empty_slot;
    if (c.capturing) {  // a graph's tables live as long as the graph (never evicted under it)
        void *d = capture_alloc(c, n * sizeof(void *));
        capture_upload(c, d, ptrs, n * sizeof(void *));
        return (const void *const *)d;
    }
    c.table_clock++;
    for (auto &e : c.tables)
        if (e.key.size() == n && std::memcmp(e.key.data(), ptrs, n * sizeof(void *)) == 0) {
            e.last_use = c.table_clock;
            return (const void *const *)e.dev;
        }
    constexpr size_t kMaxTables = 512;
    Ctx::TableEntry *slot = nullptr;
    if (c.tables.size() < kMaxTables) {
        c.tables.emplace_back();
        slot = &c.tables.back();
    } else {
        slot = &c.tables[0];
        for (auto &e : c.tables)
            if (e.last_use < slot->last_use) slot = &e;
        VR_CUDA(cudaFreeAsync(slot->dev, c.stream));  // stream-ordered: earlier users finish first
        slot->dev = nullptr;
    }
    slot->key.assign(ptrs, ptrs + n);
    slot->last_use = c.table_clock;
    VR_CUDA(cudaMallocAsync(&slot->dev, n * sizeof(void *), c.stream));
    upload_async(c, slot->dev, ptrs, n * sizeof(void *));
    return (const void *const *)slot->dev;
}

void upload_async(Ctx &c, void *dst, const void *src, size_t bytes) {
    if (c.capturing) {  // the staging ring is reused: a captured copy from it would replay stale data
        capture_upload(c, dst, src, bytes);
        return;
    }
    const char *p = (const char *)src;
    char *d = (char *)dst;
    while (bytes) {
        const size_t chunk = bytes < Ctx::kStageBytes ? bytes : Ctx::kStageBytes;
        const int slot = c.stage_next;
        c.stage_next = (c.stage_next + 1) % Ctx::kStageSlots;
        VR_CUDA(cudaEventSynchronize(c.stage_evt[slot]));  // previous copy out of this slot is done
        char *h = c.stage + (size_t)slot * Ctx::kStageBytes;
        std::memcpy(h, p, chunk);
        VR_CUDA(cudaMemcpyAsync(d, h, chunk, cudaMemcpyHostToDevice, c.stream));
        VR_CUDA(cudaEventRecord(c.stage_evt[slot], c.stream));
        p += chunk;
        d += chunk;
        bytes -= chunk;
    }
}
}

extern "C" {

const char *vr_last_error(void) { return g_err.c_str(); }
unsigned long long vr_launch_count(void) { return __atomic_load_n(&vr::g_launches, __ATOMIC_RELAXED); }

int vr_ctx_create(int log_n, int num_q, const uint64_t *primes, uint64_t seed, int sym_enc, int device, vr_ctx **out) {
    return guard([&] {
        if (log_n < 2 || log_n > 17) throw vr::VrError(VR_ERR_ENGINE, "log_n must be in [2, 17]");
        if (num_q < 1 || num_q + 1 > vr::MAXP) throw vr::VrError(VR_ERR_ENGINE, "unsupported number of primes");
        VR_CUDA(cudaSetDevice(device));
        auto *h = new vr_ctx();
        try {
        vr::Ctx &c = h->c;
        c.device = device;
        c.log_n = log_n;
        c.n = 1 << log_n;
        c.slots = c.n / 2;
        c.L = num_q - 1;
        c.np = num_q + 1;
        c.seed = seed;
        c.sym_enc = sym_enc;
        const int n = c.n, np = c.np;
        for (int p = 0; p < np; p++) {
            const uint64_t q = primes[p];
            if (q >= (1ull << 61) || q % (2ull * n) != 1)
                throw vr::VrError(VR_ERR_ENGINE, "primes must be < 2^61 and == 1 mod 2N");
            c.q[p] = q;
            u128h r = (~(u128h)0) / q;
            c.primes.m[p] = vr::Modulus{q, (uint64_t)(r >> 64), (uint64_t)r};
        }
        std::vector<ulonglong2> tw((size_t)np * n), itw((size_t)np * n);
        std::vector<double> twd((size_t)np * n), itwd((size_t)np * n);
        c.h_ntt_const.resize(np);
        for (int p = 0; p < np; p++) {
            const uint64_t q = c.q[p];
            const uint64_t psi = h_min_psi(q, n), ipsi = h_inv(psi, q);
            std::vector<uint64_t> pw(n), ipw(n);
            pw[0] = ipw[0] = 1;
            for (int i = 1; i < n; i++) { pw[i] = h_mulmod(pw[i - 1], psi, q); ipw[i] = h_mulmod(ipw[i - 1], ipsi, q); }
            for (int i = 0; i < n; i++) {
                const uint32_t r = h_brev(i, log_n);
                tw[(size_t)p * n + i] = make_ulonglong2(pw[r], h_shoup(pw[r], q));
                itw[(size_t)p * n + i] = make_ulonglong2(ipw[r], h_shoup(ipw[r], q));
                twd[(size_t)p * n + i] = (double)pw[r];
                itwd[(size_t)p * n + i] = (double)ipw[r];
            }
            const uint64_t ninv = h_inv((uint64_t)n % q, q);
            const uint64_t w0n = h_mulmod(itw[(size_t)p * n + 1].x, ninv, q);
            // FP64 path when every intermediate of a transform stays an exact integer below 2^51
            // (|values| <= 16 q through 14 forward stages); VR_NTT_F64=0 keeps every prime integer.
            static const bool f64_on = [] {
                const char *e = getenv("VR_NTT_F64");
                return e == nullptr || atoi(e) != 0;
            }();
            const int f64 = (f64_on && q < (1ull << 46)) ? 1 : 0;
            c.h_ntt_const[p] = vr::NttConst{ninv, h_shoup(ninv, q), w0n, h_shoup(w0n, q), (double)q, 1.0 / (double)q,
                                            (double)ninv, (double)w0n, f64, (double)((1ull << 32) % q)};
        }
        std::vector<uint64_t> liftk((size_t)vr::MAXP * vr::MAXP, 0), kshift(vr::MAXP, 0);
        for (int a = 0; a < np; a++) kshift[a] = c.q[a] * (((1ull << 47) + c.q[a] - 1) / c.q[a]);
        for (int a = 0; a < np; a++) {
            if (c.h_ntt_const[a].f64) c.f64mask |= 1ull << a;
            for (int b = 0; b < np; b++) {
                const uint64_t qa = c.q[a], qb = c.q[b];
                liftk[(size_t)a * vr::MAXP + b] = (qb - qa % qb) % qb;  // == qb * ceil(qa / qb) - qa
            }
        }
        c.h_inv_tab.assign((size_t)np * np * 2, 0);
        for (int a = 0; a < np; a++)
            for (int b = 0; b < np; b++) {
                if (a == b) continue;
                const uint64_t v = h_inv(c.q[a] % c.q[b], c.q[b]);
                c.h_inv_tab[((size_t)a * np + b) * 2] = v;
                c.h_inv_tab[((size_t)a * np + b) * 2 + 1] = h_shoup(v, c.q[b]);
            }
        std::vector<uint64_t> rr((size_t)(c.L + 1) * vr::RR_STRIDE, 0);
        {
            const uint64_t P = c.q[np - 1];
            for (int l = 1; l <= c.L; l++) {
                uint64_t *row = rr.data() + (size_t)l * vr::RR_STRIDE;
                const uint64_t ql = c.q[l];
                for (int i = 0; i < l; i++) {
                    const uint64_t q = c.q[i], pm = P % q, pqm = h_mulmod(pm, ql % q, q), inv = h_inv(pqm, q);
                    row[i * 8 + 0] = pm;
                    row[i * 8 + 1] = h_shoup(pm, q);
                    row[i * 8 + 2] = pqm;
                    row[i * 8 + 3] = inv;
                    row[i * 8 + 4] = h_shoup(inv, q);
                }
                const uint64_t pq = P % ql, pinv = h_inv(pq, ql);
                row[vr::MAXP * 8 + 0] = pq;
                row[vr::MAXP * 8 + 1] = h_shoup(pq, ql);
                row[vr::MAXP * 8 + 2] = pinv;
                row[vr::MAXP * 8 + 3] = h_shoup(pinv, ql);
                row[vr::MAXP * 8 + 4] = P;
            }
        }
        std::vector<double> zr(n), zi(n);
        for (int k = 0; k < n; k++) {
            const double ang = M_PI * (double)k / (double)n;
            zr[k] = cos(ang);
            zi[k] = sin(ang);
        }
        // per-stage twiddles for the slot FFT: stage with half-length hs, butterfly j uses zeta^(4 j S / (2 hs))
        std::vector<double> ftw(2 * (size_t)c.slots, 0.0);
        for (int hs = 1; hs < c.slots; hs <<= 1)
            for (int j = 0; j < hs; j++) {
                const size_t idx = (size_t)4 * j * (c.slots / (2 * hs));
                ftw[2 * (hs + j)] = zr[idx];
                ftw[2 * (hs + j) + 1] = zi[idx];
            }
        std::vector<int> sp(c.slots);
        uint64_t g = 1;
        for (int j = 0; j < c.slots; j++) { sp[j] = (int)((g - 1) / 4); g = (g * 5) % (2ull * n); }
        std::vector<int> ps(c.slots);
        {
            int logS = 0;
            while ((1 << logS) < c.slots) logS++;
            for (int j = 0; j < c.slots; j++) {
                unsigned x = (unsigned)sp[j], r = 0;
                for (int b = 0; b < logS; b++) r |= ((x >> b) & 1u) << (logS - 1 - b);
                ps[r] = j;
            }
        }
        std::vector<uint64_t> cdt(vr::CDT_LEN);
        build_cdt(cdt.data());

        c.tw2 = upload(c, tw);
        c.itw2 = upload(c, itw);
        c.twd = upload(c, twd);
        c.liftk = upload(c, liftk);
        c.kshift = upload(c, kshift);
        c.itwd = upload(c, itwd);
        c.ntt_const = upload(c, c.h_ntt_const);
        c.inv_tab = upload(c, c.h_inv_tab);
        c.rr_tab = upload(c, rr);
        c.zr = upload(c, zr);
        c.zi = upload(c, zi);
        c.ftw = upload(c, ftw);
        c.slot_pos = upload(c, sp);
        c.pos_slot = upload(c, ps);
        c.cdt = upload(c, cdt);
        VR_CUDA(cudaStreamCreateWithFlags(&c.own, cudaStreamNonBlocking));
        c.stream = c.own;  // until vr_set_stream installs the caller's stream
        VR_CUDA(cudaStreamCreateWithFlags(&c.aux, cudaStreamNonBlocking));
        VR_CUDA(cudaStreamCreateWithFlags(&c.side, cudaStreamNonBlocking));
        VR_CUDA(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming));
        VR_CUDA(cudaEventCreateWithFlags(&c.ev_join, cudaEventDisableTiming));
        {
            int least = 0, greatest = 0;
            VR_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            VR_CUDA(cudaStreamCreateWithPriority(&c.hi, cudaStreamNonBlocking, greatest));
        }
        VR_CUDA(cudaEventCreateWithFlags(&c.ev_hi, cudaEventDisableTiming));
        VR_CUDA(cudaEventCreateWithFlags(&c.ev_hi_done, cudaEventDisableTiming));
        VR_CUDA(cudaMallocHost((void **)&c.stage, (size_t)vr::Ctx::kStageSlots * vr::Ctx::kStageBytes));
        for (int i = 0; i < vr::Ctx::kStageSlots; i++)
            VR_CUDA(cudaEventCreateWithFlags(&c.stage_evt[i], cudaEventDisableTiming));
        {
            // keep freed scratch in the stream-ordered pool instead of returning it at every sync
            cudaMemPool_t pool;
            VR_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
            uint64_t thr = ~0ull;
            VR_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        }
        vr::keygen(c);
        VR_CUDA(cudaStreamSynchronize(c.stream));
        } catch (...) {
            destroy_ctx(h);  // no partially built context (device tables, streams, keys) leaks
            throw;
        }
        *out = h;
    });
}

int vr_ctx_destroy(vr_ctx *h) {
    if (!h) return VR_OK;
    return guard([&] { destroy_ctx(h); });
}

// Move the context to stream s: the current scratch arena is parked under its stream and s gets
// its own (Ctx::parked), so a call on one stream never reuses bytes another may still touch.
static void set_stream(vr::Ctx &c, cudaStream_t s) {
    if (s == c.stream) return;
    vr::Ctx::ArenaState &old = c.parked[c.stream];
    old.arena = c.arena;
    old.cap = c.arena_cap;
    old.top = c.arena_top;
    old.peak = c.arena_peak;
    old.big_free = std::move(c.big_free);
    vr::Ctx::ArenaState cur;
    auto it = c.parked.find(s);
    if (it != c.parked.end()) {
        cur = std::move(it->second);
        c.parked.erase(it);
    }
    c.arena = cur.arena;
    c.arena_cap = cur.cap;
    c.arena_top = cur.top;
    c.arena_peak = cur.peak;
    c.big_free = std::move(cur.big_free);
    c.stream = s;
}

int vr_set_stream(vr_ctx *h, void *stream) {
    // NULL is the legacy default stream (torch's default stream); the private stream is kept
    // for vr_ctx_destroy either way.
    return guard([&] { set_stream(h->c, (cudaStream_t)stream); });
}

int vr_fork_stream(vr_ctx *h, void *stream) {
    // `stream` waits for everything queued on the context's stream, then becomes the context's stream
    // (vr_set_stream switches back).  Lets a caller run a call on a side stream -- e.g. the deferred
    // encryption of a product's operands on the slot stream that will run the product.
    return guard([&] {
        vr::Ctx &c = h->c;
        const cudaStream_t s = (cudaStream_t)stream;
        if (s == c.stream) return;
        VR_CUDA(cudaEventRecord(c.ev_fork, c.stream));
        VR_CUDA(cudaStreamWaitEvent(s, c.ev_fork, 0));
        set_stream(c, s);
    });
}

int vr_sync(vr_ctx *h) {
    return guard([&] { VR_CUDA(cudaStreamSynchronize(h->c.stream)); });
}

int vr_gen_relin_key(vr_ctx *h) {
    return guard([&] { vr::relin_key(h->c); });
}

int vr_galois_elt(vr_ctx *h, int64_t steps, uint32_t *g_out) {
    return guard([&] {
        const int64_t S = h->c.slots;
        uint64_t e = (uint64_t)(((steps % S) + S) % S);
        const uint64_t m = 2ull * h->c.n;
        uint64_t g = 1, b = 5 % m;  // 5^e mod 2N by squaring (the rotation hot path asks for many)
        while (e) {
            if (e & 1) g = g * b % m;
            b = b * b % m;
            e >>= 1;
        }
        *g_out = (uint32_t)g;
    });
}

int vr_gen_galois_key(vr_ctx *h, uint32_t g) {
    return guard([&] { vr::galois_key(h->c, g); });
}

static void export_dev(vr::Ctx &c, const uint64_t *d, size_t words, uint64_t *host) {
    VR_CUDA(cudaMemcpyAsync(host, d, words * 8, cudaMemcpyDeviceToHost, c.stream));
    VR_CUDA(cudaStreamSynchronize(c.stream));
}

int vr_export_secret(vr_ctx *h, uint64_t *host_out) {
    return guard([&] { export_dev(h->c, h->c.s_ntt, (size_t)h->c.np * h->c.n, host_out); });
}
int vr_export_public_key(vr_ctx *h, uint64_t *host_out) {
    return guard([&] { export_dev(h->c, h->c.pk, (size_t)2 * (h->c.L + 1) * h->c.n, host_out); });
}
int vr_export_relin_key(vr_ctx *h, uint64_t *host_out) {
    return guard([&] { export_dev(h->c, vr::relin_key(h->c), h->c.key_words(), host_out); });
}
int vr_export_galois_key(vr_ctx *h, uint32_t g, uint64_t *host_out) {
    return guard([&] { export_dev(h->c, vr::galois_key(h->c, g), h->c.key_words(), host_out); });
}

int vr_ntt(vr_ctx *h, uint64_t *data, int polys, int limbs, int prime0, int inverse) {
    return guard([&] {
        vr::Ctx &c = h->c;
        if (prime0 < 0 || prime0 + limbs > c.np) throw vr::VrError(VR_ERR_ENGINE, "prime index out of range");
        vr::NttBatch b{data, polys * limbs, limbs, (long long)limbs * c.n, limbs, prime0, 0, 0};
        if (inverse) vr::ntt_inverse(c, b);
        else vr::ntt_forward(c, b);
    });
}

int vr_encode(vr_ctx *h, const double *vals, int count, int nvals, int level, double scale, uint64_t *pt_out) {
    return guard([&] {
        check_level(h->c, level);
        if (nvals > h->c.slots) throw vr::VrError(VR_ERR_CAPACITY, "payload exceeds slot count");
        if (count > 0) vr::encode_plain(h->c, vals, count, nvals, level, scale, pt_out);
    });
}

int vr_encode_coeffs(vr_ctx *h, const double *vals, int count, int nvals, double scale, int64_t *m_out) {
    return guard([&] {
        if (nvals > h->c.slots) throw vr::VrError(VR_ERR_CAPACITY, "payload exceeds slot count");
        if (count > 0) vr::encode_coeffs(h->c, vals, count, nvals, scale, m_out);
    });
}

int vr_encrypt(vr_ctx *h, const double *vals, int count, int nvals, int level, double scale, uint64_t nonce0, uint64_t *ct_out) {
    return guard([&] {
        check_level(h->c, level);
        if (nvals > h->c.slots) throw vr::VrError(VR_ERR_CAPACITY, "payload exceeds slot count");
        if (count > 0) vr::encrypt(h->c, vals, count, nvals, level, scale, nonce0, ct_out);
    });
}

int vr_encrypt_strided(vr_ctx *h, const double *src, long long sc, long long s1, long long s2, int p, int nvals, int count,
                       int level, double scale, uint64_t nonce0, uint64_t *ct_out) {
    return guard([&] {
        check_level(h->c, level);
        if (nvals > h->c.slots) throw vr::VrError(VR_ERR_CAPACITY, "payload exceeds slot count");
        if (count > 0) vr::encrypt_src(h->c, src, sc, s1, s2, p, nvals, count, level, scale, nonce0, ct_out);
    });
}

int vr_encrypt_strided2(vr_ctx *h, const double *src0, long long sc0, long long s1_0, long long s2_0, int p0, int nvals0,
                        int count0, uint64_t *ct0, const double *src1, long long sc1, long long s1_1, long long s2_1, int p1,
                        int nvals1, int count1, uint64_t *ct1, int level, double scale, uint64_t nonce0) {
    return guard([&] {
        check_level(h->c, level);
        if (nvals0 > h->c.slots || nvals1 > h->c.slots) throw vr::VrError(VR_ERR_CAPACITY, "payload exceeds slot count");
        if (count0 <= 0 || count1 <= 0) throw vr::VrError(VR_ERR_ENGINE, "both batches must be non-empty");
        vr::encrypt_src2(h->c, src0, sc0, s1_0, s2_0, p0, nvals0, count0, ct0, src1, sc1, s1_1, s2_1, p1, nvals1, count1, ct1,
                         level, scale, nonce0);
    });
}

// Host-array forms of the strided encryptions: the raw matrix is staged through the context's
// pinned ring into stream-ordered scratch (one cudaMemcpyAsync per 64 KB) and encrypted by the
// same launches, so a caller holding plain host arrays needs no device buffers of its own.
int vr_encrypt_strided_host(vr_ctx *h, const double *host, long long len, long long off, long long sc, long long s1,
                            long long s2, int p, int nvals, int count, int level, double scale, uint64_t nonce0,
                            uint64_t *ct_out) {
    return guard([&] {
        vr::Ctx &c = h->c;
        check_level(c, level);
        if (nvals > c.slots) throw vr::VrError(VR_ERR_CAPACITY, "payload exceeds slot count");
        if (len <= 0 || off < 0 || off >= len) throw vr::VrError(VR_ERR_ENGINE, "empty host source");
        if (count <= 0) return;
        vr::Scratch d(c, sizeof(double) * (size_t)len);
        vr::upload_async(c, d.p, host, sizeof(double) * (size_t)len);
        vr::encrypt_src(c, d.as<double>() + off, sc, s1, s2, p, nvals, count, level, scale, nonce0, ct_out);
    });
}

int vr_encrypt_strided2_host(vr_ctx *h, const double *host0, long long len0, long long off0, long long sc0, long long s1_0,
                             long long s2_0, int p0, int nvals0, int count0, uint64_t *ct0, const double *host1,
                             long long len1, long long off1, long long sc1, long long s1_1, long long s2_1, int p1, int nvals1,
                             int count1, uint64_t *ct1, int level, double scale, uint64_t nonce0) {
    return guard([&] {
        vr::Ctx &c = h->c;
        check_level(c, level);
        if (nvals0 > c.slots || nvals1 > c.slots) throw vr::VrError(VR_ERR_CAPACITY, "payload exceeds slot count");
        if (count0 <= 0 || count1 <= 0) throw vr::VrError(VR_ERR_ENGINE, "both batches must be non-empty");
        if (len0 <= 0 || len1 <= 0 || off0 < 0 || off1 < 0 || off0 >= len0 || off1 >= len1)
            throw vr::VrError(VR_ERR_ENGINE, "empty host source");
        vr::Scratch d0(c, sizeof(double) * (size_t)len0), d1(c, sizeof(double) * (size_t)len1);
        vr::upload_async(c, d0.p, host0, sizeof(double) * (size_t)len0);
        vr::upload_async(c, d1.p, host1, sizeof(double) * (size_t)len1);
        vr::encrypt_src2(c, d0.as<double>() + off0, sc0, s1_0, s2_0, p0, nvals0, count0, ct0, d1.as<double>() + off1, sc1, s1_1,
                         s2_1, p1, nvals1, count1, ct1, level, scale, nonce0);
    });
}

// Decode without blocking the host: decrypt + decode on `stream` (NULL: the context stream), copy
// the [count][S] doubles into the ticket's pinned buffer and record its completion event.  The
// ciphertext metadata travels as one staged upload (pointers | scales | degrees | levels).
int vr_decode_submit(vr_ctx *h, const uint64_t *const *cts, const int *degs, const int *levels, const double *scales,
                     int count, void *stream, int *ticket) {
    return guard([&] {
        vr::Ctx &c = h->c;
        *ticket = -1;
        if (count <= 0) throw vr::VrError(VR_ERR_ENGINE, "nothing to decode");
        int id = -1;
        for (int i = 0; i < (int)c.tickets.size() && id < 0; i++)
            if (!c.tickets[i].busy) id = i;
        if (id < 0) {
            if (c.tickets.size() >= 256) throw vr::VrError(VR_ERR_ENGINE, "too many decodes in flight (vr_decode_wait releases one)");
            c.tickets.emplace_back();
            id = (int)c.tickets.size() - 1;
        }
        const size_t bytes = sizeof(double) * (size_t)count * c.slots;
        {
            vr::Ctx::DecodeTicket &tk = c.tickets[id];
            if (tk.cap < bytes) {
                if (tk.host) cudaFreeHost(tk.host);
                tk.host = nullptr;
                tk.cap = 0;
                VR_CUDA(cudaHostAlloc((void **)&tk.host, bytes, cudaHostAllocDefault));
                tk.cap = bytes;
            }
            if (!tk.done) VR_CUDA(cudaEventCreateWithFlags(&tk.done, cudaEventDisableTiming));
        }
        struct Restore {
            vr::Ctx &c;
            cudaStream_t caller;
            ~Restore() { set_stream(c, caller); }
        } restore{c, c.stream};
        const cudaStream_t s = stream ? (cudaStream_t)stream : c.stream;
        set_stream(c, s);
        const size_t n = (size_t)count, off_s = 8 * n, off_d = 16 * n, off_l = 20 * n, total = 24 * n;
        std::vector<char> blob(total);
        std::memcpy(blob.data(), cts, 8 * n);
        std::memcpy(blob.data() + off_s, scales, 8 * n);
        std::memcpy(blob.data() + off_d, degs, 4 * n);
        std::memcpy(blob.data() + off_l, levels, 4 * n);
        vr::Scratch meta(c, total), out(c, bytes);
        vr::upload_async(c, meta.p, blob.data(), total);
        const char *m = (const char *)meta.p;
        vr::decrypt_decode(c, (const uint64_t *const *)m, (const int *)(m + off_d), (const int *)(m + off_l),
                           (const double *)(m + off_s), count, out.as<double>(), nullptr);
        vr::Ctx::DecodeTicket &tk = c.tickets[id];
        VR_CUDA(cudaMemcpyAsync(tk.host, out.p, bytes, cudaMemcpyDeviceToHost, s));
        VR_CUDA(cudaEventRecord(tk.done, s));
        tk.bytes = bytes;
        tk.busy = true;
        *ticket = id;
    });
}

int vr_decode_wait(vr_ctx *h, int ticket, double *host_out) {
    return guard([&] {
        vr::Ctx &c = h->c;
        if (ticket < 0 || ticket >= (int)c.tickets.size() || !c.tickets[ticket].busy)
            throw vr::VrError(VR_ERR_ENGINE, "unknown decode ticket");
        vr::Ctx::DecodeTicket &tk = c.tickets[ticket];
        VR_CUDA(cudaEventSynchronize(tk.done));
        if (host_out) std::memcpy(host_out, tk.host, tk.bytes);
        tk.busy = false;
    });
}

int vr_decrypt_decode(vr_ctx *h, const uint64_t *const *cts, const int *degs, const int *levels, const double *scales,
                      int count, double *out, int64_t *coeffs_out) {
    return guard([&] {
        if (count <= 0) return;
        vr::Ctx &c = h->c;
        vr::PtrTable t(c, vec(cts, count));
        vr::DevArray<int> dd(c, degs, count), dl(c, levels, count);
        vr::DevArray<double> ds(c, scales, count);
        vr::decrypt_decode(c, t.c_(), dd.get(), dl.get(), ds.get(), count, out, coeffs_out);
    });
}

int vr_add(vr_ctx *h, const uint64_t *const *a, const uint64_t *const *b, uint64_t *const *out, int count, int deg, int level,
           int op) {
    return guard([&] {
        check_level(h->c, level);
        if (count <= 0) return;
        vr::Ctx &c = h->c;
        vr::PtrTable ta(c, vec(a, count)), tb(c, vec(b, count)), to(c, vecm(out, count));
        vr::binop(c, ta.c_(), tb.c_(), to.m_(), count, deg + 1, level + 1, op);
    });
}

int vr_tensor(vr_ctx *h, const uint64_t *const *a, const uint64_t *const *b, uint64_t *const *out, int count, int level) {
    return guard([&] {
        check_level(h->c, level);
        if (count <= 0) return;
        vr::Ctx &c = h->c;
        vr::PtrTable ta(c, vec(a, count)), tb(c, vec(b, count)), to(c, vecm(out, count));
        vr::tensor(c, ta.c_(), tb.c_(), to.m_(), count, level + 1);
    });
}

int vr_relin(vr_ctx *h, const uint64_t *const *d3, uint64_t *const *out, int count, int level) {
    return guard([&] {
        check_level(h->c, level);
        if (count <= 0) return;
        vr::Ctx &c = h->c;
        vr::PtrTable ti(c, vec(d3, count)), to(c, vecm(out, count));
        vr::relin_batch(c, ti.c_(), to.m_(), count, level);
    });
}

int vr_rescale(vr_ctx *h, const uint64_t *const *in, uint64_t *const *out, int count, int deg, int level) {
    return guard([&] {
        check_level(h->c, level);
        if (level < 1) throw vr::VrError(VR_ERR_ENGINE, "multiplicative depth exhausted (level 0)");
        if (count <= 0) return;
        vr::Ctx &c = h->c;
        vr::PtrTable ti(c, vec(in, count)), to(c, vecm(out, count));
        vr::rescale(c, ti.c_(), to.m_(), count, deg + 1, level);
    });
}

int vr_relin_rescale(vr_ctx *h, const uint64_t *const *d3, uint64_t *const *out, int count, int level) {
    return guard([&] {
        check_level(h->c, level);
        if (level < 1) throw vr::VrError(VR_ERR_ENGINE, "multiplicative depth exhausted (level 0)");
        if (count <= 0) return;
        vr::Ctx &c = h->c;
        vr::PtrTable ti(c, vec(d3, count)), to(c, vecm(out, count));
        vr::relin_rescale_batch(c, ti.c_(), to.m_(), count, level);
    });
}

int vr_mul(vr_ctx *h, const uint64_t *const *a, const uint64_t *const *b, uint64_t *const *out, int count, int level) {
    return guard([&] {
        check_level(h->c, level);
        if (level < 1) throw vr::VrError(VR_ERR_ENGINE, "multiplicative depth exhausted (level 0)");
        if (count <= 0) return;
        vr::Ctx &c = h->c;
        vr::PtrTable ta(c, vec(a, count)), tb(c, vec(b, count)), to(c, vecm(out, count));
        vr::mul_batch(c, ta.c_(), tb.c_(), to.m_(), count, level);
    });
}

int vr_mul_plain(vr_ctx *h, const uint64_t *const *ct, const uint64_t *const *pt, uint64_t *const *out, int count, int deg,
                 int level, int shared_pt) {
    return guard([&] {
        check_level(h->c, level);
        if (count <= 0) return;
        vr::Ctx &c = h->c;
        vr::PtrTable ta(c, vec(ct, count)), tp(c, vec(pt, shared_pt ? 1 : count)), to(c, vecm(out, count));
        vr::mul_plain(c, ta.c_(), tp.c_(), to.m_(), count, deg + 1, level + 1, shared_pt);
    });
}

int vr_mul_scalar(vr_ctx *h, const uint64_t *const *ct, int64_t s, uint64_t *const *out, int count, int deg, int level) {
    return guard([&] {
        check_level(h->c, level);
        if (count <= 0) return;
        vr::Ctx &c = h->c;
        vr::PtrTable ta(c, vec(ct, count)), to(c, vecm(out, count));
        vr::mul_scalar(c, ta.c_(), to.m_(), count, deg + 1, level + 1, vr::limb_scalars(c, s, level + 1));
    });
}

int vr_add_const(vr_ctx *h, uint64_t *const *ct, int64_t s, int count, int level) {
    return guard([&] {
        check_level(h->c, level);
        if (count <= 0) return;
        vr::Ctx &c = h->c;
        vr::PtrTable ta(c, vecm(ct, count));
        vr::add_const(c, ta.m_(), count, level + 1, vr::limb_scalars(c, s, level + 1));
    });
}

int vr_drop_level(vr_ctx *h, const uint64_t *const *in, uint64_t *const *out, int count, int deg, int level_from, int level_to) {
    return guard([&] {
        check_level(h->c, level_from);
        if (level_to < 0 || level_to > level_from) throw vr::VrError(VR_ERR_ENGINE, "bad target level");
        if (count <= 0) return;
        vr::Ctx &c = h->c;
        vr::PtrTable ta(c, vec(in, count)), to(c, vecm(out, count));
        vr::copy_limbs(c, ta.c_(), to.m_(), count, deg + 1, level_from + 1, level_to + 1, 0);
    });
}

int vr_rotate(vr_ctx *h, const uint64_t *const *in, uint64_t *const *out, int count, int level, int nrot, const int64_t *steps) {
    return guard([&] {
        check_level(h->c, level);
        if (count <= 0 || nrot <= 0) return;
        vr::Ctx &c = h->c;
        std::vector<uint32_t> gs(nrot);
        for (int r = 0; r < nrot; r++) {
            uint32_t g;
            vr_galois_elt(h, steps[r], &g);
            gs[r] = g;
        }
        vr::PtrTable ta(c, vec(in, count)), to(c, vecm(out, (size_t)count * nrot));
        vr::rotate_batch(c, ta.c_(), to.m_(), count, level, nrot, gs.data());
    });
}

int vr_keyswitch(vr_ctx *h, const uint64_t *poly, int level, uint32_t g, uint64_t *out) {
    return guard([&] {
        check_level(h->c, level);
        vr::Ctx &c = h->c;
        const uint64_t *key = g == 0 ? vr::relin_key(c) : vr::galois_key(c, g);
        vr::PtrTable tp(c, std::vector<const uint64_t *>{poly}), to(c, std::vector<const uint64_t *>{out});
        vr::keyswitch_poly(c, tp.c_(), 1, level, key, to.m_());
    });
}

int vr_bench_butterflies(vr_ctx *h, int blocks, int iters, uint64_t *d_sink) {
    return guard([&] { vr::bfly_peak(h->c, blocks, iters, d_sink); });
}

int vr_bench_butterflies_f64(vr_ctx *h, int blocks, int iters, uint64_t *d_sink) {
    return guard([&] { vr::bfly_peak_f64(h->c, blocks, iters, d_sink); });
}

int vr_mod_reduce(vr_ctx *h, uint64_t *data, long long polys, int level) {
    return guard([&] {
        check_level(h->c, level);
        if (polys > 0) vr::mod_fixup(h->c, data, polys, level + 1);
    });
}

int vr_matmul_outer(vr_ctx *h, const uint64_t *const *L, const uint64_t *const *R, int n, int nb, int level, uint64_t *const *out) {
    return guard([&] {
        check_level(h->c, level);
        if (level < 1) throw vr::VrError(VR_ERR_ENGINE, "multiplicative depth exhausted (level 0)");
        if (n <= 0) throw vr::VrError(VR_ERR_LAYOUT, "matmul_outer needs at least one column ciphertext");
        vr::Ctx &c = h->c;
        std::vector<uintptr_t> key{1, (uintptr_t)n, (uintptr_t)nb, (uintptr_t)level};
        key.insert(key.end(), (const uintptr_t *)L, (const uintptr_t *)L + (size_t)n * nb);
        key.insert(key.end(), (const uintptr_t *)R, (const uintptr_t *)R + n);
        key.insert(key.end(), (const uintptr_t *)out, (const uintptr_t *)out + nb);
        auto body = [&] {
            vr::PtrTable tl(c, vec(L, (size_t)n * nb)), tr(c, vec(R, n)), to(c, vecm(out, nb));
            vr::matmul_outer(c, tl.c_(), tr.c_(), n, nb, level, to.m_());
        };
        // Small products (config 1: 4 MB of operands, ~20 us of device work) are bound by the host
        // submitting nine launches on three streams: replay them as one CUDA graph from the second
        // call on.  Large ones stay eager: the device is the bottleneck there, and eager launches
        // keep the programmatic overlap of one call's first kernel with the previous call's tail
        // (cfg 2: 80.4 us/step eager vs 88.1 as a graph, tools/step_probe.py).
        const size_t operand_bytes = (size_t)(nb + 1) * n * 2 * (level + 1) * c.n * 8;
        if (operand_bytes <= vr::graph_max_bytes()) vr::run_graphed(c, std::move(key), body);
        else body();
    });
}

int vr_matmul_outer_many(vr_ctx *h, const uint64_t *const *L, const uint64_t *const *R, int n, int count, int level,
                         uint64_t *const *out) {
    return guard([&] {
        check_level(h->c, level);
        if (level < 1) throw vr::VrError(VR_ERR_ENGINE, "multiplicative depth exhausted (level 0)");
        if (n <= 0) throw vr::VrError(VR_ERR_LAYOUT, "matmul_outer needs at least one column ciphertext");
        if (count <= 0) return;
        if (count > 4096) throw vr::VrError(VR_ERR_LAYOUT, "matmul_outer_many: at most 4096 products per call");
        vr::Ctx &c = h->c;
        std::vector<uintptr_t> key{3, (uintptr_t)n, (uintptr_t)count, (uintptr_t)level};
        key.insert(key.end(), (const uintptr_t *)L, (const uintptr_t *)L + (size_t)n * count);
        key.insert(key.end(), (const uintptr_t *)R, (const uintptr_t *)R + (size_t)n * count);
        key.insert(key.end(), (const uintptr_t *)out, (const uintptr_t *)out + count);
        auto body = [&] {
            vr::PtrTable tl(c, vec(L, (size_t)n * count)), tr(c, vec(R, (size_t)n * count)), to(c, vecm(out, count));
            vr::matmul_outer_many(c, tl.c_(), tr.c_(), n, count, level, to.m_());
        };
        // launch-bound by construction (that is what the batch is for): replayed as one CUDA graph
        const size_t pair_bytes = (size_t)2 * n * 2 * (level + 1) * c.n * 8;  // one product's operands
        if (pair_bytes <= vr::graph_max_bytes()) vr::run_graphed(c, std::move(key), body);
        else body();
    });
}

int vr_matmul_outer_async(vr_ctx *h, const uint64_t *const *L, const uint64_t *const *R, int n, int nb, int level,
                          uint64_t *const *out, void **slot_stream) {
    return guard([&] {
        *slot_stream = nullptr;
        check_level(h->c, level);
        if (level < 1) throw vr::VrError(VR_ERR_ENGINE, "multiplicative depth exhausted (level 0)");
        if (n <= 0) throw vr::VrError(VR_ERR_LAYOUT, "matmul_outer needs at least one column ciphertext");
        *slot_stream = (void *)vr::matmul_outer_async(h->c, L, R, n, nb, level, out);
    });
}

int vr_async_slot(vr_ctx *h, void **slot_stream) {
    return guard([&] { *slot_stream = (void *)vr::next_async_slot(h->c); });
}

int vr_join(vr_ctx *h) {
    return guard([&] {
        vr::Ctx &c = h->c;
        for (cudaStream_t s : c.slot_stream) {
            if (!s) continue;
            VR_CUDA(cudaEventRecord(c.ev_join, s));
            VR_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
        }
    });
}

// ---- ciphertexts owned through the C-ABI ------------------------------------------------------
int vr_ct_alloc(vr_ctx *h, int level, int degree, double scale, vr_ct **out) {
    return guard([&] {
        *out = nullptr;
        check_level(h->c, level);
        if (degree < 1 || degree > 2) throw vr::VrError(VR_ERR_ENGINE, "degree must be 1 or 2");
        auto *ct = new vr_ct();
        ct->level = level;
        ct->degree = degree;
        ct->scale = scale;
        const cudaError_t e = cudaMalloc((void **)&ct->data, sizeof(uint64_t) * (degree + 1) * (level + 1) * h->c.n);
        if (e != cudaSuccess) {
            cudaGetLastError();
            delete ct;
            throw vr::VrError(VR_ERR_CUDA, std::string("vr_ct_alloc: ") + cudaGetErrorString(e));
        }
        *out = ct;
    });
}

int vr_ct_free(vr_ctx *h, vr_ct *ct) {
    if (!ct) return VR_OK;
    return guard([&] {
        VR_CUDA(cudaStreamSynchronize(h->c.stream));  // no queued work may still touch it
        cudaFree(ct->data);
        delete ct;
    });
}

uint64_t *vr_ct_data(const vr_ct *ct) { return ct ? ct->data : nullptr; }
int vr_ct_level(const vr_ct *ct) { return ct ? ct->level : -1; }
int vr_ct_degree(const vr_ct *ct) { return ct ? ct->degree : -1; }
double vr_ct_scale(const vr_ct *ct) { return ct ? ct->scale : 0.0; }

static size_t ct_words(const vr::Ctx &c, const vr_ct *ct) { return (size_t)(ct->degree + 1) * (ct->level + 1) * c.n; }

int vr_ct_upload(vr_ctx *h, vr_ct *ct, const uint64_t *host) {
    return guard([&] {
        VR_CUDA(cudaMemcpyAsync(ct->data, host, ct_words(h->c, ct) * 8, cudaMemcpyHostToDevice, h->c.stream));
        VR_CUDA(cudaStreamSynchronize(h->c.stream));
    });
}

int vr_ct_download(vr_ctx *h, const vr_ct *ct, uint64_t *host) {
    return guard([&] {
        VR_CUDA(cudaMemcpyAsync(host, ct->data, ct_words(h->c, ct) * 8, cudaMemcpyDeviceToHost, h->c.stream));
        VR_CUDA(cudaStreamSynchronize(h->c.stream));
    });
}

int vr_encrypt_host(vr_ctx *h, const double *host_vals, int count, int nvals, double scale, uint64_t nonce0,
                    vr_ct *const *cts) {
    return guard([&] {
        vr::Ctx &c = h->c;
        if (nvals > c.slots) throw vr::VrError(VR_ERR_CAPACITY, "payload exceeds slot count");
        if (count <= 0) return;
        for (int i = 0; i < count; i++)
            if (cts[i]->level != c.L || cts[i]->degree != 1) throw vr::VrError(VR_ERR_ENGINE, "fresh ciphertexts are degree 1 at the top level");
        const int w = nvals > 0 ? nvals : 1;
        vr::Scratch vals(c, sizeof(double) * count * w), outs(c, sizeof(uint64_t) * count * 2 * (c.L + 1) * c.n);
        if (nvals > 0) VR_CUDA(cudaMemcpyAsync(vals.p, host_vals, sizeof(double) * count * nvals, cudaMemcpyHostToDevice, c.stream));
        vr::encrypt(c, vals.as<double>(), count, nvals, c.L, scale, nonce0, outs.as<uint64_t>());
        const size_t words = (size_t)2 * (c.L + 1) * c.n;
        for (int i = 0; i < count; i++) {
            VR_CUDA(cudaMemcpyAsync(cts[i]->data, outs.as<uint64_t>() + i * words, words * 8, cudaMemcpyDeviceToDevice, c.stream));
            cts[i]->scale = scale;
        }
        VR_CUDA(cudaStreamSynchronize(c.stream));  // the host buffer may be released on return
    });
}

int vr_decrypt_host(vr_ctx *h, const vr_ct *const *cts, int count, double *host_out) {
    return guard([&] {
        vr::Ctx &c = h->c;
        if (count <= 0) return;
        std::vector<const uint64_t *> ptrs(count);
        std::vector<int> degs(count), lvls(count);
        std::vector<double> scl(count);
        for (int i = 0; i < count; i++) {
            ptrs[i] = cts[i]->data;
            degs[i] = cts[i]->degree;
            lvls[i] = cts[i]->level;
            scl[i] = cts[i]->scale;
        }
        vr::Scratch out(c, sizeof(double) * count * c.slots);
        {
            vr::PtrTable t(c, ptrs);
            vr::DevArray<int> dd(c, degs.data(), count), dl(c, lvls.data(), count);
            vr::DevArray<double> ds(c, scl.data(), count);
            vr::decrypt_decode(c, t.c_(), dd.get(), dl.get(), ds.get(), count, out.as<double>(), nullptr);
        }
        VR_CUDA(cudaMemcpyAsync(host_out, out.p, sizeof(double) * count * c.slots, cudaMemcpyDeviceToHost, c.stream));
        VR_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int vr_matmul_outer_ct(vr_ctx *h, const vr_ct *const *L, const vr_ct *const *R, int n, int nb, vr_ct *const *out) {
    return guard([&] {
        vr::Ctx &c = h->c;
        if (n <= 0 || nb < 1 || nb > 4 || nb == 3) throw vr::VrError(VR_ERR_LAYOUT, "matmul_outer needs n >= 1 and 1, 2 or 4 row blocks");
        const int level = R[0]->level;
        const double ls = L[0]->scale, rs = R[0]->scale;
        for (int i = 0; i < nb * n; i++)
            if (L[i]->level != level || L[i]->degree != 1 || L[i]->scale != ls) throw vr::VrError(VR_ERR_LAYOUT, "left operands differ in level/scale/degree");
        for (int i = 0; i < n; i++)
            if (R[i]->level != level || R[i]->degree != 1 || R[i]->scale != rs) throw vr::VrError(VR_ERR_LAYOUT, "right operands differ in level/scale/degree");
        if (level < 1) throw vr::VrError(VR_ERR_ENGINE, "multiplicative depth exhausted (level 0)");
        for (int b = 0; b < nb; b++)
            if (out[b]->level != level - 1 || out[b]->degree != 1) throw vr::VrError(VR_ERR_LAYOUT, "outputs must be degree 1 at level - 1");
        std::vector<const uint64_t *> lp(nb * n), rp(n), op(nb);
        for (int i = 0; i < nb * n; i++) lp[i] = L[i]->data;
        for (int i = 0; i < n; i++) rp[i] = R[i]->data;
        for (int b = 0; b < nb; b++) op[b] = out[b]->data;
        vr::PtrTable tl(c, lp), tr(c, rp), to(c, op);
        vr::matmul_outer(c, tl.c_(), tr.c_(), n, nb, level, to.m_());
        for (int b = 0; b < nb; b++) out[b]->scale = ls * rs / (double)c.q[level];
    });
}

// ---- multi-GPU: native NCCL communicator --------------------------------------------------------
int vr_comm_unique_id(void *id_out) {
    return guard([&] { vr::comm_unique_id(id_out); });
}

int vr_comm_init(vr_ctx *h, const void *id, int rank, int nranks) {
    return guard([&] { vr::comm_init(h->c, id, rank, nranks); });
}

int vr_comm_destroy(vr_ctx *h) {
    return guard([&] { vr::comm_destroy(h->c); });
}

int vr_sum_partials(vr_ctx *h, uint64_t *data, long long polys, int level, int root) {
    return guard([&] {
        check_level(h->c, level);
        if (root >= h->c.nranks) throw vr::VrError(VR_ERR_ENGINE, "root rank out of range");
        vr::sum_partials(h->c, data, polys, level, root);
    });
}

int vr_tensor_sum(vr_ctx *h, const uint64_t *const *L, const uint64_t *const *R, int n, int nb, int level, uint64_t *const *out) {
    return guard([&] {
        check_level(h->c, level);
        if (n <= 0) throw vr::VrError(VR_ERR_LAYOUT, "tensor_sum needs at least one column ciphertext");
        vr::Ctx &c = h->c;
        vr::PtrTable tl(c, vec(L, (size_t)n * nb)), tr(c, vec(R, n)), to(c, vecm(out, nb));
        vr::tensor_sum(c, tl.c_(), tr.c_(), n, nb, level + 1, to.m_());
    });
}

int vr_tensor_sum_mode(vr_ctx *h, const uint64_t *const *L, const uint64_t *const *R, int n, int level, uint64_t *out, int mode) {
    return guard([&] {
        check_level(h->c, level);
        if (n <= 0) throw vr::VrError(VR_ERR_LAYOUT, "tensor_sum needs at least one column ciphertext");
        if (mode != 1 && mode != 2) throw vr::VrError(VR_ERR_ENGINE, "mode must be 1 (d2) or 2 (d0, d1)");
        vr::Ctx &c = h->c;
        vr::PtrTable tl(c, vec(L, n)), tr(c, vec(R, n)), to(c, std::vector<const uint64_t *>{out});
        vr::tensor_sum_mode(c, tl.c_(), tr.c_(), n, 1, level + 1, to.m_(), mode);
    });
}

int vr_conv_columns(vr_ctx *h, const uint64_t *const *X, int C, int W, int k, const int64_t *w, const uint64_t *bias, int F,
                    const int *out_cols, int nout, const uint64_t *mask_pt, int level, uint64_t *const *Y) {
    return guard([&] {
        check_level(h->c, level);
        if (level < 1) throw vr::VrError(VR_ERR_ENGINE, "multiplicative depth exhausted (level 0)");
        if (k < 1 || C < 1 || F < 1 || W < 1) throw vr::VrError(VR_ERR_ENGINE, "bad conv shape");
        for (int o = 0; o < nout; o++)
            if (out_cols[o] < 0 || out_cols[o] + k > W) throw vr::VrError(VR_ERR_ENGINE, "output column out of range");
        std::vector<const uint64_t *> xs(X, X + (size_t)C * W);
        std::vector<uint64_t *> ys(Y, Y + (size_t)F * nout);
        vr::conv_columns(h->c, xs, C, W, k, w, bias, F, out_cols, nout, mask_pt, level, ys);
    });
}

int vr_pt_matvec(vr_ctx *h, const uint64_t *const *X, int nx, const uint64_t *const *PT, int ny, int level,
                 uint64_t *const *Y) {
    return guard([&] {
        check_level(h->c, level);
        if (level < 1) throw vr::VrError(VR_ERR_ENGINE, "multiplicative depth exhausted (level 0)");
        if (nx <= 0 || ny <= 0) return;
        vr::Ctx &c = h->c;
        vr::PtrTable tx(c, vec(X, nx)), tp(c, vec(PT, (size_t)nx * ny)), ty(c, vecm(Y, ny));
        vr::pt_matvec(c, tx.c_(), nx, tp.c_(), ny, level, ty.m_());
    });
}

int vr_poly_activation(vr_ctx *h, const uint64_t *const *x, int count, int level, const int64_t *kc, int c3_zero,
                       uint64_t *const *out) {
    return guard([&] {
        check_level(h->c, level);
        if (level < 2) throw vr::VrError(VR_ERR_ENGINE, "multiplicative depth exhausted (poly_activation needs 2 levels)");
        if (count <= 0) return;
        vr::Ctx &c = h->c;
        vr::PtrTable tx(c, vec(x, count)), to(c, vecm(out, count));
        vr::poly_activation(c, tx.c_(), count, level, kc, c3_zero, to.m_());
    });
}

}  // extern "C"
