// dslash_h16.cu -- the EO dslash kernels for h16 storage, 12-real links (dslash_impl.cuh).
#include "dslash_impl.cuh"

namespace qdpb {
int dslash_h16(qdp_ctx ctx, const DslashArgs &a) { return dslash_t<h16, 12>(ctx, a); }
}  // namespace qdpb
