// dslash_f18.cu -- the EO dslash kernels for float storage, 18-real links (dslash_impl.cuh).
#include "dslash_impl.cuh"

namespace qdpb {
int dslash_f18(qdp_ctx ctx, const DslashArgs &a) { return dslash_t<float, 18>(ctx, a); }
}  // namespace qdpb
