"""Expression texts for qdp_jit_eval (include/qdpb.h, "run-time generated site expressions")."""


def hopping(gauge: str = "$0", psi: str = "$1", grouped: bool = True, literal: bool = False) -> str:
    """The hopping term of PAPER.md:282 (section VIII-C),
        sum_mu (1 - gamma_mu) U_mu(x) psi(x + mu) + (1 + gamma_mu) U_mu(x - mu)^dag psi(x - mu),
    with shift() as in Fig. 1.  The generator pairs every term A with a term
    +-gamma_mu A into a spin projection (1320 flop/site), whatever the grouping (grouped: each
    (1 -/+ gamma_mu) A in parentheses; otherwise one flat sum).  literal: A written as 1*(A), which
    defeats the pairing, so the sum is evaluated as written (2664 flop/site with the 1* scalings) --
    for comparison."""
    terms = []
    for m in range(4):
        f = f"{gauge}[{m}]*shift({psi},{m},+1)"
        b = f"shift(adj({gauge}[{m}])*{psi},{m},-1)"
        fa, ba = (f"1*({f})", f"1*({b})") if literal else (f, b)
        if grouped:
            terms.append(f"({fa} - gamma({m})*({f})) + ({ba} + gamma({m})*{b})")
        else:
            terms.append(f"{fa} - gamma({m})*({f}) + {ba} + gamma({m})*{b}")
    return " + ".join(terms)
