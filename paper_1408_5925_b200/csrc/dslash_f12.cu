// dslash_f12.cu -- the EO dslash kernels for float storage, 12-real links (dslash_impl.cuh).
#include "dslash_impl.cuh"

namespace qdpb {
int dslash_f12(qdp_ctx ctx, const DslashArgs &a) { return dslash_t<float, 12>(ctx, a); }
}  // namespace qdpb
