"""Expression texts for qdp_jit_eval (include/qdpb.h, "run-time generated site expressions")."""


def hopping(gauge: str = "$0", psi: str = "$1", grouped: bool = True) -> str:
    """The hopping term of PAPER.md:282 (section VIII-C),
        sum_mu (1 - gamma_mu) U_mu(x) psi(x + mu) + (1 + gamma_mu) U_mu(x - mu)^dag psi(x - mu),
    with shift() as in Fig. 1.  grouped: every (1 -/+ gamma_mu) A in parentheses,
    which the generator turns into a spin projection (1320 flop/site); otherwise the sum is evaluated
    literally (each U psi product still formed once)."""
    terms = []
    for m in range(4):
        f = f"{gauge}[{m}]*shift({psi},{m},+1)"
        b = f"shift(adj({gauge}[{m}])*{psi},{m},-1)"
        if grouped:
            terms.append(f"({f} - gamma({m})*({f})) + ({b} + gamma({m})*{b})")
        else:
            terms.append(f"{f} - gamma({m})*({f}) + {b} + gamma({m})*{b}")
    return " + ".join(terms)
