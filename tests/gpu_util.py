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
