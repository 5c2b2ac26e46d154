// graph.cu -- CUDA-graph cache of fixed-shape drivers (see graph.cuh).
#include <algorithm>
#include <map>
#include <mutex>

#include "encode.cuh"
#include "graph.cuh"
#include "ring.cuh"

namespace vr {

bool graphs_enabled() {
    static const bool on = [] {
        const char *e = getenv("VR_GRAPH");
        return e == nullptr || atoi(e) != 0;
    }();
    return on;
}

size_t graph_max_bytes() {
    static const size_t v = [] {
        const char *e = getenv("VR_GRAPH_MAX_MB");
        return (size_t)((e ? atof(e) : 32.0) * 1048576.0);
    }();
    return v;
}

void *capture_alloc(Ctx &c, size_t bytes) {
    void *p = nullptr;
    VR_CUDA(cudaMallocAsync(&p, bytes, c.side));
    c.capturing->blocks.push_back(p);
    return p;
}

void capture_upload(Ctx &c, void *dst, const void *src, size_t bytes) {
    // synchronous w.r.t. the host buffer (it may be a temporary), off the capturing stream
    VR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c.side));
    VR_CUDA(cudaStreamSynchronize(c.side));
}

static void free_mem(Ctx &c, GraphMem &m) {
    for (void *p : m.blocks) cudaFreeAsync(p, c.side);
    m.blocks.clear();
    cudaStreamSynchronize(c.side);
    cudaGetLastError();
}

static void release(Ctx &c, GraphEntry &g) {
    if (g.exec) {
        cudaDeviceSynchronize();  // the graph may still be running on whichever stream launched it
        cudaGraphExecDestroy(g.exec);
        g.exec = nullptr;
    }
    if (g.graph) {
        cudaGraphDestroy(g.graph);
        g.graph = nullptr;
    }
    free_mem(c, g.mem);
}

void graphs_release(Ctx &c) {
    for (auto &g : c.graphs) release(c, g);
    c.graphs.clear();
}

GraphEntry *graph_lookup(Ctx &c, std::vector<uintptr_t> &&key) {
    c.graph_clock++;
    for (auto &g : c.graphs)
        if (g.key == key) {
            g.last_use = c.graph_clock;
            return &g;
        }
    constexpr size_t kMaxGraphs = 32;  // 8 slots x 2 forms x 2 shapes
    if (c.graphs.size() >= kMaxGraphs) {
        auto it = std::min_element(c.graphs.begin(), c.graphs.end(),
                                   [](const GraphEntry &a, const GraphEntry &b) { return a.last_use < b.last_use; });
        release(c, *it);
        c.graphs.erase(it);
    }
    c.graphs.emplace_back();
    GraphEntry &g = c.graphs.back();
    g.key = std::move(key);
    g.last_use = c.graph_clock;
    return &g;
}

void graph_capture_begin(Ctx &c, GraphEntry &g, cudaStream_t &user, unsigned long long &k0) {
    user = c.stream;
    k0 = __atomic_load_n(&g_launches, __ATOMIC_RELAXED);
    // record on the private non-blocking stream (the legacy default stream cannot be captured);
    // the replay is ordered on the caller's stream
    VR_CUDA(cudaStreamBeginCapture(c.own, cudaStreamCaptureModeRelaxed));
    c.stream = c.own;
    c.capturing = &g.mem;
}

void graph_capture_abort(Ctx &c, GraphEntry &g, cudaStream_t user, unsigned long long k0) {
    cudaGraph_t graph = nullptr;
    cudaStreamEndCapture(c.own, &graph);
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    c.capturing = nullptr;
    c.stream = user;
    __atomic_store_n(&g_launches, k0, __ATOMIC_RELAXED);
    free_mem(c, g.mem);
    g.seen = -1000000;  // never try to capture this key again
}

void graph_capture_end(Ctx &c, GraphEntry &g, cudaStream_t user, unsigned long long k0, bool keep_graph) {
    c.capturing = nullptr;
    c.stream = user;
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(c.own, &graph);
    const unsigned long long k1 = __atomic_load_n(&g_launches, __ATOMIC_RELAXED);
    g.kernels = k1 - k0;
    __atomic_fetch_sub(&g_launches, g.kernels, __ATOMIC_RELAXED);  // recorded, not launched
    if (e != cudaSuccess) {
        cudaGetLastError();
        if (graph) cudaGraphDestroy(graph);
        free_mem(c, g.mem);
        throw VrError(4, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e));
    }
    VR_CUDA(cudaStreamSynchronize(c.side));  // capture-time allocations and uploads are complete
    const cudaError_t ei = cudaGraphInstantiateWithFlags(&g.exec, graph, cudaGraphInstantiateFlagUseNodePriority);
    if (keep_graph && ei == cudaSuccess) g.graph = graph;  // its nodes stay addressable for SetParams
    else cudaGraphDestroy(graph);
    if (ei != cudaSuccess) {
        cudaGetLastError();
        g.exec = nullptr;
        free_mem(c, g.mem);
        throw VrError(4, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ei));
    }
}

void graph_launch(Ctx &c, GraphEntry &g) {
    VR_CUDA(cudaGraphLaunch(g.exec, c.stream));
    __atomic_fetch_add(&g_launches, g.kernels, __ATOMIC_RELAXED);
}

// Slot streams are process-wide per device and never destroyed: tensors recorded on them (the
// caching allocator's record_stream of operands and outputs) may outlive the context that ran the
// product, and the allocator records events on the stream when such a tensor is freed.
static cudaStream_t slot_stream(int device, int k) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, cudaStream_t> pool;
    std::lock_guard<std::mutex> lock(mu);
    cudaStream_t &s = pool[{device, k}];
    if (!s) {
        int cur = device;
        VR_CUDA(cudaGetDevice(&cur));
        if (cur != device) VR_CUDA(cudaSetDevice(device));
        const cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        if (cur != device) cudaSetDevice(cur);
        if (e != cudaSuccess) {
            cudaGetLastError();
            s = nullptr;
            throw VrError(4, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
        }
    }
    return s;
}

// Kernel node at the head of every asynchronous slot graph: writes the operand and output pointer
// tables the recorded driver reads.  Its parameters (the pointers themselves) are replaced before
// every replay, so one recorded graph per (slot, shape) serves any operands and any output buffer.
__global__ void k_set_tables(SetTables a) {
    for (int i = threadIdx.x; i < a.count; i += blockDim.x) a.dst[i] = const_cast<uint64_t *>(a.p[i]);
}

static SetTables make_tables(uint64_t **dst, const uint64_t *const *L, const uint64_t *const *R, uint64_t *const *out, int n,
                             int nb) {
    SetTables a;
    a.dst = dst;
    a.count = (nb + 1) * n + nb;
    int k = 0;
    for (int i = 0; i < nb * n; i++) a.p[k++] = L[i];
    for (int i = 0; i < n; i++) a.p[k++] = R[i];
    for (int i = 0; i < nb; i++) a.p[k++] = out[i];
    return a;
}

cudaStream_t next_async_slot(Ctx &c) {
    const int k = c.slot_next;
    if (!c.slot_stream[k]) c.slot_stream[k] = slot_stream(c.device, k);
    return c.slot_stream[k];
}

// Asynchronous matmul_outer.  Calls rotate over the slot streams; slot k replays its own graph of the
// one-pass form (one (d0, d1, d2) tensor sum, then the relinearise+rescale chain) recorded with
// graph-owned scratch, so the latency-bound chain of one call overlaps the streaming sums of the next
// ones.  The slot stream first waits for everything already queued on the caller's stream (the
// operands); the caller orders any later use of the output after the returned stream (the Python
// layer makes its current stream wait before the result is read, and records the operand tensors on
// it for the caching allocator).  The graph is keyed by (slot, shape, level) only: its pointer tables
// are written by its first node, whose parameters carry this call's pointers.  The first call of a
// key runs synchronously and the second records the graph.  Slots swept on B200 (cfg 2, 200
// products): synchronous 80.4 us per product; 2 slots 74.5, 3 57.4, 4 51.7, 5 49.3, 6 47.0,
// 8 45.3 (20 products: 68.7 at 3 slots, 59.2 at 8).
cudaStream_t matmul_outer_async(Ctx &c, const uint64_t *const *L, const uint64_t *const *R, int n, int nb, int level,
                                uint64_t *const *out) {
    auto sync_body = [&] {
        PtrTable tl(c, std::vector<const uint64_t *>(L, L + (size_t)n * nb)), tr(c, std::vector<const uint64_t *>(R, R + n)),
            to(c, std::vector<const uint64_t *>(out, out + nb));
        matmul_outer(c, tl.c_(), tr.c_(), n, nb, level, to.m_());
    };
    // A caller may have produced the operands ON the slot stream this call was going to use (the
    // deferred encryptions of encode_left / encode_right run there, vr_fork_stream): when the product
    // runs synchronously on the context stream instead, that stream first waits for the slot.
    auto sync_after_slot = [&] {
        const cudaStream_t s = next_async_slot(c);
        VR_CUDA(cudaEventRecord(c.ev_join, s));
        VR_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
        sync_body();
    };
    if (!graphs_enabled() || nb > 4 || (nb + 1) * n + nb > kSetMaxPtrs) {
        sync_after_slot();
        return nullptr;
    }
    const int k = c.slot_next;
    // Two recorded forms per (slot, shape, level).  Resident operands: every chain transform as one
    // cluster kernel (7 kernels per product instead of 9: the overlapped chains are dispatch-bound).
    // Operands encrypted since the previous product (an encrypt -> product -> decode loop): the two-pass
    // transforms, whose independent CTAs slip between the clusters of the next product's 5,120-CTA
    // encryption NTT where 8-CTA clusters would queue behind them (e2e 4.4k vs 4.1k HE matmul/s).
    const bool fresh_operands = c.enc_calls != c.enc_seen;
    c.enc_seen = c.enc_calls;
    const uintptr_t form = fresh_operands ? 0 : 1;
    GraphEntry *g = graph_lookup(c, std::vector<uintptr_t>{2, (uintptr_t)k, (uintptr_t)n, (uintptr_t)nb, (uintptr_t)level, form});
    if (!g->exec) {
        if (g->seen < 1) {
            g->seen++;
            sync_after_slot();
            return nullptr;
        }
        relin_key(c);  // generated outside any capture
        cudaStream_t user;
        unsigned long long k0;
        graph_capture_begin(c, *g, user, k0);
        c.capture_cl = form == 1;
        try {
            // one contiguous graph-owned block: L table, R table, out table
            auto **tabs = (uint64_t **)capture_alloc(c, sizeof(void *) * ((nb + 1) * n + nb));
            g->out_table = tabs;
            const SetTables first = make_tables(tabs, L, R, out, n, nb);
            // the tensor sum carries the pointers in its own parameters when it can (one kernel less per
            // product: the overlapped chains are dispatch-bound); else a one-block kernel writes the tables
            g->ts_first = tensor_sum_takes_params(nb) && n >= 1;
            if (g->ts_first) {
                c.ts_params = &first;
                c.ts_node = nullptr;
            } else {
                k_set_tables<<<1, 256, 0, c.stream>>>(first);
                check_launch("k_set_tables");
                cudaStreamCaptureStatus cs;
                const cudaGraphNode_t *deps = nullptr;
                size_t nd = 0;
                VR_CUDA(cudaStreamGetCaptureInfo(c.stream, &cs, nullptr, nullptr, &deps, &nd));
                if (nd != 1) throw VrError(4, "matmul_outer_async: unexpected capture dependencies");
                g->out_node = deps[0];
            }
            matmul_outer(c, (const uint64_t *const *)tabs, (const uint64_t *const *)(tabs + (size_t)nb * n), n, nb, level,
                         tabs + (size_t)(nb + 1) * n, true);
            if (g->ts_first) {
                if (c.ts_params || !c.ts_node) throw VrError(4, "matmul_outer_async: the tensor sum did not take its pointer parameters");
                g->out_node = c.ts_node;
            }
        } catch (...) {
            c.capture_cl = false;
            c.ts_params = nullptr;
            graph_capture_abort(c, *g, user, k0);
            throw;
        }
        c.capture_cl = false;
        graph_capture_end(c, *g, user, k0, true);
        if (g->ts_first) VR_CUDA(cudaGraphKernelNodeGetParams(g->out_node, &g->ts_kp));  // the graph is kept: its storage stays valid
    } else {
        SetTables a = make_tables(g->out_table, L, R, out, n, nb);
        if (g->ts_first) {
            // k_tensor_sum_ldp(SetTables, n, nl, N, primes, O, rb): replace the first parameter only
            void *args[7];
            for (int i = 0; i < 7; i++) args[i] = g->ts_kp.kernelParams[i];
            args[0] = &a;
            cudaKernelNodeParams kp = g->ts_kp;
            kp.kernelParams = args;
            kp.extra = nullptr;
            VR_CUDA(cudaGraphExecKernelNodeSetParams(g->exec, g->out_node, &kp));
        } else {
            void *args[] = {&a};
            cudaKernelNodeParams kp = {};
            kp.func = (void *)k_set_tables;
            kp.gridDim = dim3(1);
            kp.blockDim = dim3(256);
            kp.sharedMemBytes = 0;
            kp.kernelParams = args;
            kp.extra = nullptr;
            VR_CUDA(cudaGraphExecKernelNodeSetParams(g->exec, g->out_node, &kp));
        }
    }
    cudaStream_t s = next_async_slot(c);
    VR_CUDA(cudaEventRecord(c.ev_fork, c.stream));  // operands (and anything before) are ready
    VR_CUDA(cudaStreamWaitEvent(s, c.ev_fork, 0));
    VR_CUDA(cudaGraphLaunch(g->exec, s));
    __atomic_fetch_add(&g_launches, g->kernels, __ATOMIC_RELAXED);
    static const int nslots = [] {
        const char *e = getenv("VR_ASYNC_SLOTS");
        const int v = e ? atoi(e) : Ctx::kSlots;
        return v < 1 ? 1 : (v > Ctx::kSlots ? Ctx::kSlots : v);
    }();
    c.slot_next = (k + 1) % nslots;
    return s;
}

}  // namespace vr
