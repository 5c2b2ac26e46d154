// graph.cuh -- CUDA-graph replay of fixed-shape drivers.
//
// A driver call is identified by a key (driver id, shape, level and every device pointer it
// touches).  The first call with a key runs eagerly; the second records the driver into a CUDA
// graph on the context's private stream (scratch buffers and pointer tables are then owned by
// the graph, see Scratch / cached_table) and every later call replays that graph on the caller's
// stream with one cudaGraphLaunch: the host submits one launch instead of a chain of nine kernel
// launches and event operations on three streams.  VR_GRAPH=0 disables it.
#pragma once
#include <utility>
#include <vector>

#include "vrhe_internal.cuh"

namespace vr {

bool graphs_enabled();
// drivers whose operands exceed this many bytes run eagerly (VR_GRAPH_MAX_MB, default 32)
size_t graph_max_bytes();
GraphEntry *graph_lookup(Ctx &c, std::vector<uintptr_t> &&key);
void graph_capture_begin(Ctx &c, GraphEntry &g, cudaStream_t &user, unsigned long long &k0);
void graph_capture_abort(Ctx &c, GraphEntry &g, cudaStream_t user, unsigned long long k0);
void graph_capture_end(Ctx &c, GraphEntry &g, cudaStream_t user, unsigned long long k0, bool keep_graph = false);
void graph_launch(Ctx &c, GraphEntry &g);

template <class F>
void run_graphed(Ctx &c, std::vector<uintptr_t> &&key, F &&body) {
    if (!graphs_enabled() || c.capturing) {
        body();
        return;
    }
    GraphEntry *g = graph_lookup(c, std::move(key));
    if (!g->exec && g->seen < 1) {
        g->seen++;
        body();
        return;
    }
    if (!g->exec) {
        cudaStream_t user;
        unsigned long long k0;
        graph_capture_begin(c, *g, user, k0);
        try {
            body();
        } catch (...) {
            graph_capture_abort(c, *g, user, k0);
            throw;
        }
        graph_capture_end(c, *g, user, k0);
    }
    graph_launch(c, *g);
}

// matmul_outer as an asynchronous slot graph (vr_matmul_outer_async): returns the slot stream the
// result is produced on, or nullptr when the call ran synchronously on c.stream
cudaStream_t next_async_slot(Ctx &c);  // the slot stream the next asynchronous call will use
cudaStream_t matmul_outer_async(Ctx &c, const uint64_t *const *L, const uint64_t *const *R, int n, int nb, int level,
                                uint64_t *const *out);

}  // namespace vr
