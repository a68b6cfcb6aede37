// dslash_d18.cu -- the EO dslash kernels for double storage, 18-real links (dslash_impl.cuh).
#include "dslash_impl.cuh"

namespace qdpb {
int dslash_d18(qdp_ctx ctx, const DslashArgs &a) { return dslash_t<double, 18>(ctx, a); }
}  // namespace qdpb
