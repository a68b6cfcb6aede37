"""Build tuning variants of libqdpb.so into variants/ (development aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1408_5925_b200 import build as b  # noqa: E402

VARIANTS = {
    "base": [],
    "b128m3": ["-DQDPB_DSLASH_MAXT=128", "-DQDPB_DSLASH_MINB=3"],
    "b128m4": ["-DQDPB_DSLASH_MAXT=128", "-DQDPB_DSLASH_MINB=4"],
    "b256m2": ["-DQDPB_DSLASH_MAXT=256", "-DQDPB_DSLASH_MINB=2", "-DQDPB_DSLASH_BLOCK=256"],
    "b64m6": ["-DQDPB_DSLASH_MAXT=64", "-DQDPB_DSLASH_MINB=6", "-DQDPB_DSLASH_BLOCK=64"],
}
names = sys.argv[1:] or list(VARIANTS)
for n in names:
    lib = os.path.join(ROOT, "variants", f"libqdpb_{n}.so")
    b.build(lib=lib, extra=VARIANTS[n], obj_dir=os.path.join(ROOT, "variants", "obj_" + n), verbose=False)
    print(lib)
