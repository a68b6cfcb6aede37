// dslash_d12.cu -- the EO dslash kernels for double storage, 12-real links (dslash_impl.cuh).
#include "dslash_impl.cuh"

namespace qdpb {
int dslash_d12(qdp_ctx ctx, const DslashArgs &a) { return dslash_t<double, 12>(ctx, a); }
}  // namespace qdpb
