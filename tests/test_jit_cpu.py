"""Front end of the run-time site-expression generator (qdp_jit_source; no GPU needed): parsing,
type rules, the Table II work accounting against the values the paper prints, common-
subexpression elimination, and NVRTC compilation of the generated source for sm_100a."""
import json
import os

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def q():
    from paper_1408_5925_b200 import qdpb
    qdpb.lib()
    return qdpb


def hopping_expr(grouped=True):
    from paper_1408_5925_b200 import exprs
    return exprs.hopping(grouped=grouped)


def test_table2_accounting_matches_paper(q):
    """Flop/byte of the generated Table II kernels = the DP values printed in PAPER.md:71-79."""
    gold = json.load(open(os.path.join(HERE, "golden", "table2_flop_byte.json")))["flop_per_byte_dp"]
    C, F, S = q.QDP_COLORMATRIX, q.QDP_FERMION, q.QDP_SPINMATRIX
    cases = {"lcm": ("$0*$1", C, [C, C], 198, 432), "upsi": ("$0*$1", F, [C, F], 264, 528),
             "spmat": ("$0*$1", S, [S, S], 480, 768), "matvec": ("$0*$1 + $0*$2", F, [C, F, F], 552, 864)}
    for name, (expr, ok, kinds, flops, t2bytes) in cases.items():
        _, w = q.qdp_jit_source(expr, ok, q.QDP_F64, kinds)
        assert (w["flops"], w["table2_bytes"]) == (flops, t2bytes), name
        assert round(w["flops"] / w["table2_bytes"], 2) == round(gold[name], 2), name
        _, w32 = q.qdp_jit_source(expr, ok, q.QDP_F32, kinds)
        assert w32["flops"] == flops and w32["table2_bytes"] == t2bytes / 2
    # matvec: Table II counts U1 twice; the compulsory count reads it once
    _, w = q.qdp_jit_source("$0*$1 + $0*$2", F, q.QDP_F64, [C, F, F])
    assert w["bytes"] == (18 + 24 + 24 + 24) * 8


def test_hopping_expression_work(q):
    """A spinor sum is flattened and every pair of terms A, +-gamma_mu A (any grouping, order or
    sign) becomes a spin projection: 8 x (12 projection + 132 U x half spinor) + 7 x 24 accumulation
    = 1320 flop/site, exactly the standard hopping-term count of the hand-written kernel (DESIGN.md
    section 7).  Compulsory bytes per EO output site = the dslash's 1536 (8 links, input, output);
    for a full-lattice output each field is read once: 4 links + input + output."""
    G, F = q.QDP_GAUGE, q.QDP_FERMION
    for grouped in (True, False):
        _, w = q.qdp_jit_source(hopping_expr(grouped), F, q.QDP_F64, [G, F], out_subset=0)
        assert w["flops"] == 8 * (12 + 132) + 7 * 24 == 1320
        assert w["bytes"] == 1536
    # order and sign do not matter: gamma term first, negated pairs
    f = "$0[0]*shift($1,0,+1)"
    for e, fl in ((f"-gamma(0)*({f}) + {f}", 144), (f"-({f}) + gamma(0)*({f})", 144),
                  (f"{f} - $1 - gamma(0)*({f})", 144 + 24)):
        _, w = q.qdp_jit_source(e, F, q.QDP_F64, [G, F])
        assert w["flops"] == fl, e
    # any gamma_mu pairs with any A, e.g. (1 - gamma_y) applied to an x-hop
    _, w = q.qdp_jit_source(f"{f} - gamma(1)*({f})", F, q.QDP_F64, [G, F])
    assert w["flops"] == 144
    # no partner (the gamma term's operand is 2A, not A): literal product, scale and subtraction
    _, w = q.qdp_jit_source(f"{f} - gamma(1)*(2*({f}))", F, q.QDP_F64, [G, F])
    assert w["flops"] == 264 + 24 + 24
    _, w = q.qdp_jit_source(hopping_expr(), F, q.QDP_F64, [G, F], out_subset=-1)
    assert w["bytes"] == (4 * 18 + 24 + 24) * 8
    _, w = q.qdp_jit_source(hopping_expr(), F, q.QDP_F32, [q.QDP_GAUGE12, F], out_subset=1)
    assert w["bytes"] == (8 * 12 + 24 + 24) * 4


def test_generated_source_structure(q):
    src, _ = q.qdp_jit_source("$0[1]*shift(shift($1,1,+1),2,-1)", q.QDP_FERMION, q.QDP_F64,
                              [q.QDP_GAUGE, q.QDP_FERMION])
    assert src.count("__global__") == 1 and "qdp_jit_kernel" in src
    assert "typedef double R;" in src
    assert "n[1] = wrap_up(n[1], a.L[1]);" in src and "n[2] = wrap_down(n[2], a.L[2]);" in src
    assert "const int p1 = p ^ 0;" in src  # two hops: same parity


@pytest.mark.parametrize("bad, msg", [("$0*", "parse error"), ("$0*$1", "cannot multiply"),
                                      ("gamma(0)", "expression is a gamma"), ("$0[0]", "non-gauge"),
                                      ("shift($0,4,1)", "direction"), ("shift($0,1,2)", "sign"),
                                      ("foo($0)", "unknown function"), ("$3", "not supplied"),
                                      ("adj($0)", "adj needs"), ("$0 + 1", "cannot add"), ("($0", "expected ')'")])
def test_errors(q, bad, msg):
    with pytest.raises(q.QdpError) as e:
        q.qdp_jit_source(bad, q.QDP_FERMION, q.QDP_F64, [q.QDP_FERMION, q.QDP_FERMION])
    assert e.value.status == q.QDP_EINVAL and msg in str(e.value)


def test_gauge_needs_link_index(q):
    with pytest.raises(q.QdpError) as e:
        q.qdp_jit_source("$0*$1", q.QDP_FERMION, q.QDP_F64, [q.QDP_GAUGE, q.QDP_FERMION])
    assert "link index" in str(e.value)


@pytest.mark.parametrize("prec", [0, 1])
def test_nvrtc_compiles_for_sm100a(q, prec):
    """The generated kernels compile to sm_100a cubins with NVRTC on a machine without a GPU."""
    for expr, ok, kinds in [("$0*$1", q.QDP_COLORMATRIX, [q.QDP_COLORMATRIX] * 2),
                            (hopping_expr(), q.QDP_FERMION, [q.QDP_GAUGE12, q.QDP_FERMION]),
                            ("gamma5*$0*adj($0)", q.QDP_SPINMATRIX, [q.QDP_SPINMATRIX])]:
        src, _ = q.qdp_jit_source(expr, ok, prec, kinds, compile=True)
        assert "qdp_jit_kernel" in src


def test_sum_expressions(q):
    """Complex-scalar expressions for qdp_jit_sum: the plaquette executes 3 colour products (594)
    + a trace (4); local norms / inner products count like the BLAS kernels (48 / 96 per spinor)."""
    G, F = q.QDP_GAUGE, q.QDP_FERMION
    plaq = "real(trace($0[0]*shift($0[1],0,+1)*adj(shift($0[0],1,+1))*adj($0[1])))"
    _, w = q.qdp_jit_source(plaq, q.QDP_JIT_SUM, q.QDP_F64, [G])
    assert w["flops"] == 3 * 198 + 4
    _, w = q.qdp_jit_source("localNorm2($0)", q.QDP_JIT_SUM, q.QDP_F64, [F])
    assert w["flops"] == 48 and w["bytes"] == 192
    _, w = q.qdp_jit_source("localInnerProduct($0,$1)", q.QDP_JIT_SUM, q.QDP_F32, [F, F], compile=True)
    assert w["flops"] == 96 and w["bytes"] == 192
    for bad, msg in [("$0", "complex scalar"), ("trace($0)", "trace needs"), ("localInnerProduct($0)", "two arguments"),
                     ("real($0)", "real needs")]:
        with pytest.raises(q.QdpError) as e:
            q.qdp_jit_source(bad, q.QDP_JIT_SUM, q.QDP_F64, [F])
        assert msg in str(e.value), bad
