"""Build tuning variants of libqdpb.so into variants/ (development aid).

  python tools/build_variants.py [name ...]
Each variant is the same source compiled with extra -D tuning macros (see internal.h)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1408_5925_b200 import build as b  # noqa: E402

VARIANTS = {
    "base": [],
    "pf_off": ["-DQDPB_PF_F12=0"],  # no fp32 reconstruct-12 link prefetch
    "h16_scalar": ["-DQDPB_H16_F32X2=0"],  # 16-bit dslash with scalar fp32 arithmetic (no FFMA2)
    # occupancy sweeps per (precision, gauge storage): min resident 64-thread blocks per SM
    "occ_a": ["-DQDPB_MINB_D12=7", "-DQDPB_MINB_F18=8", "-DQDPB_MINB_F12=8"],
    "occ_b": ["-DQDPB_MINB_D12=8", "-DQDPB_MINB_F18=10", "-DQDPB_MINB_F12=10"],
    "occ_c": ["-DQDPB_MINB_D12=5", "-DQDPB_MINB_F18=12", "-DQDPB_MINB_F12=12"],
    "occ_d": ["-DQDPB_MINB_D12=4", "-DQDPB_MINB_F18=16", "-DQDPB_MINB_F12=16"],
}
names = sys.argv[1:] or list(VARIANTS)
for n in names:
    lib = os.path.join(ROOT, "variants", f"libqdpb_{n}.so")
    b.build(lib=lib, extra=VARIANTS[n], obj_dir=os.path.join(ROOT, "variants", "obj_" + n), verbose=False)
    print(lib)
