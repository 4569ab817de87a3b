"""Helpers for the -m gpu parity tests (inputs from synth, references from oracle)."""

import numpy as np

from synth.problems import stack


def have_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def make_ctx(problems, **kw):
    import torch
    from paper_2204_08057_b200 import build
    build.build()
    from paper_2204_08057_b200.kroncg import KronCG
    st = stack(problems)
    hits = torch.from_numpy(st["hits"]).cuda() if st["hits"] is not None else None
    kw.setdefault("prior", problems[0].prior)
    ctx = KronCG(problems[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"],
                 hits=hits, **kw)
    Y = torch.from_numpy(st["Y"]).cuda()
    return ctx, Y


def rel(a, b):
    a = np.asarray(a).reshape(-1)
    b = np.asarray(b).reshape(-1)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def oracle_count_envelope(fn, G, b, **kw):
    """The oracle's iteration count is itself uncertain by rounding where CG needs a number of steps
    comparable to the unknowns (measured: a 2^-50 relative change of b moves the oracle's HS count by
    up to 2, and the HS and single-pass variants differ by up to 9 -- DESIGN.md reading R34).  Returns
    (lo, hi, result on b): the counts of `fn` on b and on b (1 +- 2^-50); the bar is then
    lo - 2 <= it_gpu <= hi + 2, which is the plain +-2 wherever the count is well determined."""
    import numpy as np
    ref = fn(G, b, **kw)
    its = [ref.iterations]
    for f in (1.0 + 2.0 ** -50, 1.0 - 2.0 ** -50):
        its.append(fn(G, np.asarray(b) * f, **kw).iterations)
    return min(its), max(its), ref
