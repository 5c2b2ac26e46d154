// ntt.cu -- plain (unfused) batched NTT / INTT entry points; the kernels live
// in ntt_impl.cuh so the key-switching code can instantiate fused variants.
#include "ntt_impl.cuh"

namespace vr {

void ntt_forward(Ctx &c, const NttBatch &b) { nttk::run_fused<false>(c, b, nttk::LdPlain{}, nttk::StPlain{}); }
void ntt_inverse(Ctx &c, const NttBatch &b) { nttk::run_fused<true>(c, b, nttk::LdPlain{}, nttk::StPlain{}); }

}  // namespace vr
