"""Shared helpers for GPU-vs-oracle parity tests (test infrastructure)."""
import numpy as np
import torch

import oracle
from paper_1212_0873_b200 import pcdm

# north_star tolerances (BASELINE.json): objective within 1e-5 relative and
# ||x_gpu - x_oracle||_inf <= 1e-4 ||x_oracle||_inf (fp32 atomics reorder sums).
F_RTOL = 1e-5
X_RTOL = 1e-4


def to_host(t):
    return t.detach().cpu().numpy()


def run_both(colptr, rowidx, val, b, lam, m, tau, iters, seed=0, x0=None, first_iter=0,
             refresh_every=0, beta_override=0.0, variant="auto", device="cuda:0", sampling=None):
    """Run the CUDA path (device x) and the oracle on the same arrays.
    sampling: None (tau-nice) or a spec (kind, tau, p_b, q) handed to both sides.
    Returns dict with x_gpu, x_orc (fp64), F_gpu (library objective), F_orc, stats, res."""
    n = colptr.numel() - 1
    dev = torch.device(device)
    prob = pcdm.Problem(m, n, colptr.to(dev), rowidx.to(dev), val.to(dev), b.to(dev), lam)
    x = torch.zeros(n, dtype=torch.float32, device=dev) if x0 is None else \
        torch.as_tensor(x0, dtype=torch.float32).to(dev).clone()
    gs = None if sampling is None else pcdm.Sampling(*sampling)
    prob.run(x, tau, iters, seed=seed, first_iter=first_iter, refresh_every=refresh_every,
             beta_override=beta_override, variant=variant, sampling=gs)
    beta_gpu = prob.beta(tau) if gs is None else prob.beta_sampling(gs)
    torch.cuda.synchronize()
    stats = prob.stats()
    F_gpu = prob.objective(x)
    r_gpu = torch.empty(m, dtype=torch.float32, device=dev)
    prob.residual(r_gpu)
    omega_gpu = prob.omega
    prob.close()
    c, r, v, bb = to_host(colptr), to_host(rowidx), to_host(val), to_host(b)
    x0h = None if x0 is None else np.asarray(to_host(torch.as_tensor(x0)), dtype=np.float32).astype(np.float64)
    res = oracle.run(m, c, r, v, bb, lam, tau, iters, seed, x0=x0h, first_iter=first_iter,
                     refresh_every=refresh_every,
                     beta_override=beta_override if beta_override > 0 else None,
                     sampling=None if sampling is None else oracle.Sampling(*sampling))
    F_orc = oracle.objective(m, c, r, v, bb, lam, res.x)
    return dict(x_gpu=to_host(x).astype(np.float64), x_orc=res.x, F_gpu=F_gpu, F_orc=F_orc,
                stats=stats, res=res, r_gpu=to_host(r_gpu), omega_gpu=omega_gpu, beta_gpu=beta_gpu)


def assert_parity(out, f_rtol=F_RTOL, x_rtol=X_RTOL):
    F_gpu, F_orc = out["F_gpu"], out["F_orc"]
    assert abs(F_gpu - F_orc) <= f_rtol * abs(F_orc), (F_gpu, F_orc)
    xo, xg = out["x_orc"], out["x_gpu"]
    scale = max(np.max(np.abs(xo)), 1e-30)
    dx = np.max(np.abs(xg - xo)) if xo.size else 0.0
    assert dx <= x_rtol * scale, (dx, scale)
    assert out["omega_gpu"] == out["res"].omega
