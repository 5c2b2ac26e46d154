// comm.cu -- the multi-GPU exchange of the column-ciphertext matmul, natively:
// NCCL communicators owned by the context and the int64 sum of degree-2 partial products.
//
// Config 5a shards the k range of C = sum_k L_k (x) R_k over ranks (multicipher.py:100-102,
// PAPER.md:909).  Every rank computes its partial (d0, d1, d2) residues with vr_tensor_sum; the
// partials are summed as plain uint64 (each residue < 2^61, so up to 8 ranks cannot wrap), reduced
// mod q_i on the device, then relinearised and rescaled once -- bit-identical for any rank count.
// NCCL is resolved at run time (dlopen "libnccl.so.2": the copy torch already loaded if any, else
// the system one), so libvrhe.so has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "encode.cuh"
#include "ring.cuh"

namespace vr {
namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char *(*error_string)(ncclResult_t) = nullptr;
    std::string err;
};

const NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.err = std::string("cannot load NCCL: ") + dlerror();
            return;
        }
        api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
        api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
        api.all_reduce = (decltype(api.all_reduce))dlsym(h, "ncclAllReduce");
        api.reduce = (decltype(api.reduce))dlsym(h, "ncclReduce");
        api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
        api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
        if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.reduce || !api.comm_destroy)
            api.err = "NCCL library lacks the collective entry points";
    });
    if (!api.err.empty()) throw VrError(4, api.err);
    return api;
}

void check_nccl(ncclResult_t r, const char *what) {
    if (r != ncclSuccess) {
        const char *msg = nccl().error_string ? nccl().error_string(r) : "?";
        throw VrError(4, std::string(what) + ": " + msg);
    }
}

}  // namespace

void comm_unique_id(void *out) {
    ncclUniqueId id;
    check_nccl(nccl().get_unique_id(&id), "ncclGetUniqueId");
    memcpy(out, &id, sizeof(id));
}

void comm_init(Ctx &c, const void *id, int rank, int nranks) {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw VrError(3, "bad rank / world size");
    if (c.comm) throw VrError(3, "context already has a communicator");
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    VR_CUDA(cudaSetDevice(c.device));
    ncclComm_t comm = nullptr;
    check_nccl(nccl().comm_init_rank(&comm, nranks, uid, rank), "ncclCommInitRank");
    c.comm = comm;
    c.rank = rank;
    c.nranks = nranks;
}

void comm_destroy(Ctx &c) {
    if (!c.comm) return;
    nccl().comm_destroy((ncclComm_t)c.comm);
    c.comm = nullptr;
    c.rank = 0;
    c.nranks = 1;
}

// Sum the [polys][level+1][N] residue partials over ranks (root < 0: all-reduce, every rank gets the
// sum; else only `root` does), then reduce mod q_i where the sum landed.
void sum_partials(Ctx &c, uint64_t *data, long long polys, int level, int root) {
    const size_t words = (size_t)polys * (level + 1) * c.n;
    if (c.comm && c.nranks > 1) {
        if (c.nranks > 8) throw VrError(3, "more than 8 ranks could overflow the uint64 residue sum");
        if (root < 0)
            check_nccl(nccl().all_reduce(data, data, words, ncclUint64, ncclSum, (ncclComm_t)c.comm, c.stream), "ncclAllReduce");
        else
            check_nccl(nccl().reduce(data, data, words, ncclUint64, ncclSum, root, (ncclComm_t)c.comm, c.stream), "ncclReduce");
    }
    if (root < 0 || root == c.rank) mod_fixup(c, data, polys, level + 1);
}

}  // namespace vr
