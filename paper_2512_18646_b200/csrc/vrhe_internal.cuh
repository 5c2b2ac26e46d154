// vrhe_internal.cuh -- context, device tables and launch helpers shared by the
// CUDA translation units of libvrhe.so.  Nothing here is exported; the C-ABI
// lives in abi.cu and is declared in include/vrhe.h.
#pragma once
#include <cstdlib>
#include <exception>
#include <utility>
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <stdexcept>
#include <unordered_map>
#include <string>
#include <vector>

#include "modarith.cuh"

namespace vr {

constexpr int MAXP = 40;
constexpr int RR_STRIDE = MAXP * 8 + 8;

struct DevPrimes {
    Modulus m[MAXP];
};

// Per-prime NTT scalars: n^-1 and (psi^-1_br[1] * n^-1), each with Shoup companion.
struct NttConst {
    uint64_t ninv, ninv_sh, w0n, w0n_sh;
    // FP64-pipe transform (primes below 2^46, see ntt_impl.cuh): q, 1/q, n^-1 and w0n as doubles
    double qd, qinv, ninv_d, w0n_d;
    int f64;
    double c32;  // 2^32 mod q (centred lifts of 60-bit residues into an FP64-body prime, LdLift)
};

// Memory owned by one captured CUDA graph (graph.cu): while a driver is being captured, every
// scratch buffer and pointer table it asks for is carved here instead of the context's arena /
// table cache, so the graph's baked-in addresses stay valid for as long as the graph lives.
struct GraphMem {
    std::vector<void *> blocks;
};

// Operand and output pointers of one asynchronous matmul_outer, carried in the kernel parameters of
// the first kernel of its slot graph (replaced before every replay, so one recorded graph serves any
// operands): p = [L (nb n)] [R (n)] [out (nb)]; the kernel copies them into the graph-owned table dst
// that the later kernels of the graph read.
constexpr int kSetMaxPtrs = 240;  // (nb + 1) n + nb pointers; 2 KB of kernel parameters
struct SetTables {
    uint64_t **dst;
    int count;
    const uint64_t *p[kSetMaxPtrs];
};

struct GraphEntry {
    std::vector<uintptr_t> key;  // driver id, shape, level, then every pointer of the call
    cudaGraphExec_t exec = nullptr;
    GraphMem mem;
    unsigned long long kernels = 0;  // kernel launches the graph replays (for vr_launch_count)
    unsigned long long last_use = 0;
    int seen = 0;  // eager runs so far (a key is captured on its second occurrence)
    // asynchronous slot graphs: the kernel node that writes the output pointer table, re-pointed at
    // every replay (cudaGraphExecKernelNodeSetParams), and the graph it belongs to
    cudaGraph_t graph = nullptr;
    cudaGraphNode_t out_node = nullptr;
    uint64_t **out_table = nullptr;
    // out_node is the tensor sum itself (pointers in its parameters) rather than a table-writing kernel:
    // its recorded launch, whose first parameter is replaced before every replay
    bool ts_first = false;
    cudaKernelNodeParams ts_kp = {};
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = 0;                 // the stream every call is ordered on (vr_set_stream)
    cudaStream_t own = 0;                    // the context's private stream (default until vr_set_stream)
    cudaStream_t aux = 0;                    // second stream for intra-driver overlap
    cudaEvent_t ev_fork = 0, ev_join = 0;    // fork/join events (timing disabled)
    cudaStream_t hi = 0;                     // highest-priority stream for latency-bound chains
    cudaEvent_t ev_hi = 0, ev_hi_done = 0;
    int log_n = 0, n = 0, slots = 0, L = 0, np = 0;  // np = L + 2 (ciphertext chain + special prime)
    uint64_t q[MAXP] = {0};
    DevPrimes primes;
    uint64_t seed = 0;
    int sym_enc = 0;

    // device tables
    ulonglong2 *tw2 = nullptr, *itw2 = nullptr;  // [np][N] (twiddle, Shoup companion) psi^(br i), psi^-(br i)
    NttConst *ntt_const = nullptr;                                                 // [np]
    uint64_t *inv_tab = nullptr;  // [np][np][2]: (q_a^-1 mod q_b, shoup)
    // fused relinearise+rescale constants per level l >= 1: rr_tab + l * RR_STRIDE
    //   [i*8 + 0..5] = P mod q_i (+shoup), (P q_l) mod q_i, (P q_l)^-1 mod q_i (+shoup), 0
    //   [MAXP*8 + 0..3] = P mod q_l (+shoup), P^-1 mod q_l (+shoup)
    uint64_t *rr_tab = nullptr;
    double *zr = nullptr, *zi = nullptr;  // zeta^k, k < N
    uint64_t f64mask = 0;          // bit p: prime p runs the FP64 NTT body
    uint64_t *kshift = nullptr;    // [MAXP] q ceil(2^47 / q): signed inputs of FP64-body transforms
    uint64_t *liftk = nullptr;     // [MAXP][MAXP] centred-lift offsets for FP64 transforms (ntt_impl.cuh LdLift)
    double *twd = nullptr, *itwd = nullptr;  // NTT twiddles as doubles [np][N] (FP64-pipe transforms)
    double *ftw = nullptr;  // FFT twiddles by stage: (re, im) pairs at [hs + j], hs = 1, 2, .., S/2, j < hs
    int *slot_pos = nullptr;              // [S]
    int *pos_slot = nullptr;              // [S] slot j whose bit-reversed FFT position is p
    uint64_t *cdt = nullptr;              // [CDT_LEN]

    // keys (device)
    uint64_t *s_ntt = nullptr;  // [np][N]
    uint64_t *s_sh = nullptr;   // [np][N] Shoup companions floor(s * 2^64 / q) of s_ntt
    uint64_t *pk = nullptr;     // [2][L+1][N]
    uint64_t *rlk = nullptr;    // [L+1][2][np][N]
    std::map<uint32_t, uint64_t *> gkeys;

    // host copies of small constants
    std::vector<NttConst> h_ntt_const;
    std::vector<uint64_t> h_inv_tab;

    // pinned staging ring for small host->device uploads (pointer tables, weights):
    // pageable cudaMemcpyAsync would block the host until the stream drains.
    static constexpr int kStageSlots = 64;
    static constexpr size_t kStageBytes = 64 << 10;
    char *stage = nullptr;
    cudaEvent_t stage_evt[kStageSlots] = {};
    int stage_next = 0;

    // value-keyed cache of device pointer tables: identical tables (same pointer values) are
    // uploaded once and reused, so steady-state driver calls issue no host->device copies.
    struct TableEntry {
        std::vector<const void *> key;
        void *dev = nullptr;
        unsigned long long last_use = 0;
    };
    std::vector<TableEntry> tables;
    unsigned long long table_clock = 0;

    // stack arena for per-call scratch (LIFO, stream-ordered reuse is safe on one stream)
    char *arena = nullptr;
    size_t arena_cap = 0, arena_top = 0, arena_peak = 0;
    // free list of big scratch blocks (> 64 MB), reused in stream order; mapping fresh multi-GB
    // blocks from the pool can stall the host for hundreds of ms
    std::vector<std::pair<size_t, void *>> big_free;
    // The arena and the big-block list are reused in the order of ONE stream.  When the caller moves
    // the context to another stream (vr_set_stream), the current arena is parked under its stream and
    // the new stream gets its own, so a call on stream B never reuses bytes stream A may still touch.
    struct ArenaState {
        char *arena = nullptr;
        size_t cap = 0, top = 0, peak = 0;
        std::vector<std::pair<size_t, void *>> big_free;
    };
    std::map<cudaStream_t, ArenaState> parked;

    // CUDA-graph cache of fixed-shape drivers (graph.cu); capturing != nullptr while one records
    std::vector<GraphEntry> graphs;
    unsigned long long graph_clock = 0;
    GraphMem *capturing = nullptr;
    bool capture_cl = false;  // the graph being recorded runs every transform as one cluster kernel (graph.cu)
    // set while a slot graph is recorded: the one-pass tensor sum takes its operand pointers from these
    // parameters (and publishes the table) instead of a separate table-writing kernel; it clears the
    // pointer once it has consumed it
    const SetTables *ts_params = nullptr;
    cudaGraphNode_t ts_node = nullptr;  // the captured node of that tensor sum
    unsigned long long enc_calls = 0, enc_seen = 0;  // encryption launches, and how many the last async product had seen
    cudaStream_t side = 0;  // non-blocking helper stream for capture-time allocations and uploads
    // asynchronous drivers (vr_matmul_outer_async): calls rotate over kSlots streams (process-wide per
    // device, graph.cu), each replaying its own graph, so consecutive independent calls overlap
    static constexpr int kSlots = 8;  // VR_ASYNC_SLOTS picks how many rotate (default all 8)
    cudaStream_t slot_stream[kSlots] = {};
    int slot_next = 0;

    // asynchronous decodes (vr_decode_submit / vr_decode_wait): a pinned result buffer and a
    // completion event per ticket, reused once the ticket has been waited for
    struct DecodeTicket {
        double *host = nullptr;
        size_t cap = 0, bytes = 0;
        cudaEvent_t done = nullptr;
        bool busy = false;
    };
    std::vector<DecodeTicket> tickets;

    // multi-GPU (comm.cu): NCCL communicator of this context's rank, or null
    void *comm = nullptr;
    int rank = 0, nranks = 1;

    size_t key_words() const { return (size_t)(L + 1) * 2 * np * n; }
};

// capture-time allocation / upload into the graph being recorded (graph.cu)
void *capture_alloc(Ctx &c, size_t bytes);
void capture_upload(Ctx &c, void *dst, const void *src, size_t bytes);
// release every cached graph (context teardown)
void graphs_release(Ctx &c);

struct VrError : std::runtime_error {
    int code;
    VrError(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define VR_CUDA(call)                                                                              \
    do {                                                                                           \
        cudaError_t _e = (call);                                                                   \
        if (_e != cudaSuccess) {                                                                   \
            cudaGetLastError(); /* do not leave the error for the next check_launch */             \
            throw ::vr::VrError(4, std::string(#call) + ": " + cudaGetErrorString(_e));            \
        }                                                                                          \
    } while (0)

// number of kernels launched by this library (bench.py reports it as gpu_launches)
extern unsigned long long g_launches;

inline void check_launch(const char *what) {
    __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw VrError(4, std::string(what) + ": " + cudaGetErrorString(e));
}

// Raise kern's dynamic shared-memory limit on the context's device to at least `smem`.
// The attribute is per (device, function) and shared by every context on that device, so the
// record of what was set is process-wide, keyed by device, only ever raised, and mutex-guarded
// (one engine per worker thread is the reference's model, engine.py:170-173).  Set for any size:
// the 48 KB default covers dynamic + static shared memory together.
void ensure_smem(Ctx &c, const void *kern, size_t smem);

// Drivers that fork work onto c.aux / c.hi temporarily point c.stream at them.  This guard
// restores the caller's stream on every exit and, when unwinding after an error, joins the side
// streams back into it so scratch freed on the caller's stream is not reused under them.
struct StreamScope {
    Ctx &c;
    cudaStream_t main;
    explicit StreamScope(Ctx &cx) : c(cx), main(cx.stream) {}
    ~StreamScope() {
        c.stream = main;
        if (std::uncaught_exceptions() > 0) {
            for (cudaStream_t s : {c.aux, c.hi}) {
                if (!s) continue;
                if (cudaEventRecord(c.ev_join, s) == cudaSuccess) cudaStreamWaitEvent(main, c.ev_join, 0);
            }
            cudaGetLastError();
        }
    }
    StreamScope(const StreamScope &) = delete;
};

// Per-call scratch.  Carved LIFO out of the context's arena (kernels on the one stream
// run in order, so the next call may reuse the bytes immediately); when the arena is
// too small the request falls back to cudaMallocAsync and the arena is regrown, to the
// high-water mark, the next time it is empty.
struct Scratch {
    Ctx &c;
    void *p = nullptr;
    size_t bytes = 0;
    bool pooled = false, big = false, graph = false;
    static constexpr size_t kArenaMaxBuffer = size_t(64) << 20, kArenaMaxCap = size_t(512) << 20;
    Scratch(Ctx &cx, size_t b) : c(cx) {
        bytes = (b + 255) & ~size_t(255);
        if (!bytes) return;
        if (c.capturing) {  // recorded into a CUDA graph: the graph owns the buffer
            p = capture_alloc(c, bytes);
            graph = true;
            return;
        }
        if (bytes > kArenaMaxBuffer) {  // big buffers: cached free list (best fit within 2x)
            size_t best = (size_t)-1;
            int bi = -1;
            for (int i = 0; i < (int)c.big_free.size(); i++) {
                const size_t sz = c.big_free[i].first;
                if (sz >= bytes && sz <= 2 * bytes && sz < best) { best = sz; bi = i; }
            }
            if (bi >= 0) {
                p = c.big_free[bi].second;
                bytes = c.big_free[bi].first;
                c.big_free.erase(c.big_free.begin() + bi);
            } else {
                VR_CUDA(cudaMallocAsync(&p, bytes, c.stream));
            }
            big = true;
            return;
        }
        if (c.arena_top == 0 && c.arena_cap < c.arena_peak) {
            if (c.arena) cudaFreeAsync(c.arena, c.stream);
            c.arena = nullptr;
            c.arena_cap = 0;
            if (cudaMallocAsync((void **)&c.arena, c.arena_peak, c.stream) == cudaSuccess) c.arena_cap = c.arena_peak;
            else cudaGetLastError();
        }
        if (c.arena && c.arena_top + bytes <= c.arena_cap) {
            p = c.arena + c.arena_top;
            c.arena_top += bytes;
            pooled = true;
        } else {
            VR_CUDA(cudaMallocAsync(&p, bytes, c.stream));
        }
        const size_t want = c.arena_top + (pooled ? 0 : bytes);
        if (want > c.arena_peak && want <= kArenaMaxCap) c.arena_peak = want;
    }
    ~Scratch() {
        if (!p || graph) return;
        if (pooled) c.arena_top -= bytes;
        else if (big) c.big_free.emplace_back(bytes, p);
        else cudaFreeAsync(p, c.stream);
    }
    template <class T>
    T *as() const { return (T *)p; }
    Scratch(const Scratch &) = delete;
};

// stream-ordered host->device copy through the pinned staging ring
void upload_async(Ctx &c, void *dst, const void *src, size_t bytes);
// device copy of a pointer table, cached by value (see Ctx::tables)
const void *const *cached_table(Ctx &c, const void *const *ptrs, size_t n);

// Upload a small host array (pointer table etc.) to a stream-ordered device buffer.
template <class T>
struct DevArray {
    Scratch s;
    DevArray(Ctx &c, const T *host, size_t count) : s(c, sizeof(T) * (count ? count : 1)) {
        if (count) upload_async(c, s.p, host, sizeof(T) * count);
    }
    T *get() const { return s.as<T>(); }
};

// ---------------------------------------------------------------------------
// NTT batch descriptor: transform t lives at
//   data + (t / group) * gstride + (t % group) * N
// and uses prime index  r < nq ? poff + r : pspecial   (r = t % group).
// skip_diag > 0 skips transforms with r == (t / group) % skip_diag (ModUp digit's own prime).
struct NttBatch {
    uint64_t *data;
    int count;
    int group;
    long long gstride;
    int nq;
    int poff;
    int pspecial;
    int skip_diag;
    // optional second segment: transforms t >= split (a multiple of group) live at data2 instead
    // (two separately allocated ciphertext batches encrypted by one launch)
    uint64_t *data2 = nullptr;
    int split = 0x7fffffff;
};

inline NttBatch batch_limbs(uint64_t *data, int polys, int limbs, int n) {
    return NttBatch{data, polys * limbs, limbs, (long long)limbs * n, limbs, 0, 0, 0};
}

void ntt_forward(Ctx &c, const NttBatch &b);
void ntt_inverse(Ctx &c, const NttBatch &b);

// grid helper
// Programmatic dependent launch (sm_90+).  A kernel started through launch_pdl may become
// resident while its predecessor on the stream is still draining; it must execute pdl_wait()
// (griddepcontrol.wait: full completion + visibility of the predecessor grid) before touching
// global memory.  pdl_trigger() lets the successor launch early.  VR_PDL=0 disables the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("VR_PDL");
        return e == nullptr || atoi(e) != 0;
    }();
    return on;
}

// Execution priority of every kernel except the streaming tensor sums: when independent products
// overlap (asynchronous matmul_outer slots), the block scheduler places the CTAs of the small
// latency-bound key-switch kernels ahead of the pending CTAs of another product's tensor sum instead
// of behind them.  Recorded graphs keep it per node (cudaGraphInstantiateFlagUseNodePriority).
// VR_CHAIN_PRIO=1 enables (default off: the tensor sums then wait behind every chain kernel and the
// cfg-2 step grows from 43 to 51 us).  Returns 0 (the default, lowest priority) when off.
inline int chain_priority() {
    static const int p = [] {
        const char *e = getenv("VR_CHAIN_PRIO");
        if (!e || atoi(e) == 0) return 0;  // off by default: measured slower (cfg 2: 43 -> 51 us per product)
        int least = 0, greatest = 0;
        if (cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        return greatest;
    }();
    return p;
}
// appends the priority attribute to at[n]; returns the new attribute count
inline unsigned add_priority_attr(cudaLaunchAttribute *at, unsigned n) {
    const int p = chain_priority();
    if (p == 0) return n;
    at[n].id = cudaLaunchAttributePriority;
    at[n].val.priority = p;
    return n + 1;
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[2];
    unsigned n = 0;
    if (pdl_enabled()) {
        at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[n].val.programmaticStreamSerializationAllowed = 1;
        n++;
    }
    cfg.attrs = at;
    cfg.numAttrs = add_priority_attr(at, n);
    VR_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

inline unsigned nblocks(long long work, int per_block) { return (unsigned)((work + per_block - 1) / per_block); }

}  // namespace vr
