// dslash.cu -- dispatch of the fused even-odd Wilson hopping term (section
// VIII-C) to its per-(precision, gauge storage) translation units (dslash_impl.cuh).
#include "internal.h"

namespace qdpb {

int dslash(qdp_ctx ctx, int prec, const DslashArgs &a) {
  if (a.h16) return dslash_h16(ctx, a);
  if (a.rec12) return prec == QDP_F64 ? dslash_d12(ctx, a) : dslash_f12(ctx, a);
  return prec == QDP_F64 ? dslash_d18(ctx, a) : dslash_f18(ctx, a);
}

}  // namespace qdpb
