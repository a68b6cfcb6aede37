// slots.h -- per-site complex "slot" map of fermion and gauge fields: slot k of the site
// (parity p, cb) lives at data + off[p][k] + cb * step[k] (2 reals of the field precision).
// Used by the layout conversion (layout.cu) and by shift (shift.cu).
#pragma once
#include "internal.h"

namespace qdpb {
struct SlotMap {
  int n;                  // 12 (fermion) or 36 (gauge: mu*9 + 3*row + col)
  long long off[2][36];   // -1: parity not present in the field
  int step[36];
  unsigned char pair[36]; // 1: slots k, k+1 are the two halves of one 16-byte element (fp32)
};
SlotMap make_slot_map(int kind, int prec, int stride, int subset);
}  // namespace qdpb
