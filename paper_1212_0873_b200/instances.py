"""Seeded synthetic LASSO instances shaped like the paper's workloads.

This module only builds INPUTS (A in CSC, b, lambda, the planted x*); it holds
none of the method's arithmetic and is the one module both the CUDA path's
tests/bench and the oracle's tests draw from ("Input recipe").

Recipe (BASELINE.json ``configs``), standing in for the
paper's 10^9-variable instance of Sec. 8.1, whose
"modified primal-dual generator" and 350 GB size are not reproducible here:

  G1  each column gets ``c`` distinct rows, uniform or Zipf(s) over rows
      (P(row = j-1) ~ j^-s, hot rows at low indices), sorted ascending;
  G2  values iid N(0,1), fp32, in sorted-row order;
  G3  x* has ``s_star`` distinct uniform positions with N(0,1) values;
  G4  b = fp32(A x* (fp64 accumulation) + 0.01 * eps), eps iid N(0,1);
  G5  lambda = 0.1 * max_i |a_i^T b| (fp64, on the fp32 b);
  G6  x0 = 0.

Randomness comes from a ``torch.Generator`` seeded with ``seed`` on
``device``; an instance is a deterministic function of (config, seed, device
type).  Parity tests always hand the SAME arrays to both sides.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import torch


@dataclasses.dataclass(frozen=True)
class InstanceConfig:
    name: str
    m: int
    n: int
    nnz_per_col: int
    s_star: int
    rows: str = "uniform"      # "uniform" | "zipf"
    zipf_s: float = 1.1
    noise: float = 0.01
    lam_frac: float = 0.1
    tau: int = 1
    iters: int = 1
    # column lengths: "fixed" (nnz_per_col each) or "pareto": len = min(len_max,
    # floor(len_min * U^(-1/alpha))), U uniform on (0, 1] -- a power-law (Zipf-tail)
    # mix of short columns and a few very long ones, like the feature columns of the
    # paper's KDDB data; nnz_per_col is then only the nominal mean
    col_lengths: str = "fixed"
    len_alpha: float = 1.5
    len_min: int = 7
    len_max: int = 10_000


# BASELINE.json "configs", in order.
CONFIGS = {
    "tiny": InstanceConfig("tiny", 2000, 1000, 10, 100, tau=32, iters=2000),
    "medium": InstanceConfig("medium", 100_000, 100_000, 20, 1000, tau=1024, iters=10_000),
    "skewed": InstanceConfig("skewed", 1_000_000, 1_000_000, 20, 10_000, rows="zipf",
                             tau=1 << 12, iters=10_000),
    "large": InstanceConfig("large", 2_000_000, 10_000_000, 20, 10_000, tau=65536, iters=2000),
    "huge": InstanceConfig("huge", 100_000_000, 500_000_000, 10, 100_000, tau=1 << 18, iters=500),
}
# Ragged column lengths (not a BASELINE.json config): the `large`
# shape with power-law column lengths (Pareto alpha = 1.5 from 7, capped at 10^4
# entries: mean ~20, ~190 columns at the cap), a stand-in for the KDDB-shaped
# feature columns of PAPER.md:1388-1392.
RAGGED_CONFIGS = {
    "ragged": InstanceConfig("ragged", 2_000_000, 10_000_000, 20, 10_000, tau=65536, iters=2000,
                             col_lengths="pareto"),
    "ragged_small": InstanceConfig("ragged_small", 20_000, 6_000, 20, 200, tau=256, iters=400,
                                   col_lengths="pareto", len_alpha=0.9, len_min=2, len_max=12_000),
}
SKEWED_TAUS = [1 << e for e in range(8, 17)]


@dataclasses.dataclass
class Instance:
    cfg: InstanceConfig
    m: int
    n: int
    colptr: torch.Tensor   # int64[n+1]
    rowidx: torch.Tensor   # int32[nnz]
    val: torch.Tensor      # float32[nnz]
    b: torch.Tensor        # float32[m]
    lam: float
    xstar_idx: torch.Tensor
    xstar_val: torch.Tensor

    @property
    def nnz(self) -> int:
        return int(self.rowidx.numel())

    def to(self, device) -> "Instance":
        return dataclasses.replace(
            self, colptr=self.colptr.to(device), rowidx=self.rowidx.to(device),
            val=self.val.to(device), b=self.b.to(device),
            xstar_idx=self.xstar_idx.to(device), xstar_val=self.xstar_val.to(device))

    def numpy(self):
        """Host numpy views (colptr, rowidx, val, b) for the oracle."""
        return (self.colptr.cpu().numpy(), self.rowidx.cpu().numpy(),
                self.val.cpu().numpy(), self.b.cpu().numpy())


def _zipf_cdf(m: int, s: float, device) -> torch.Tensor:
    j = torch.arange(1, m + 1, dtype=torch.float64, device=device)
    w = j.pow(-s)
    cdf = torch.cumsum(w, 0)
    return cdf / cdf[-1]


def _draw_rows(k: int, c: int, m: int, gen, device, zipf_cdf: Optional[torch.Tensor]):
    """k columns x c distinct rows each, sorted ascending (G1), int64."""
    def fresh(count):
        if zipf_cdf is None:
            return torch.randint(0, m, (count,), generator=gen, device=device, dtype=torch.int64)
        u = torch.rand(count, generator=gen, device=device, dtype=torch.float64)
        return torch.searchsorted(zipf_cdf, u, right=True).clamp_(max=m - 1)

    rows = fresh(k * c).view(k, c)
    rows, _ = torch.sort(rows, dim=1)
    while True:
        dup = torch.zeros_like(rows, dtype=torch.bool)
        dup[:, 1:] = rows[:, 1:] == rows[:, :-1]
        nd = int(dup.sum())
        if nd == 0:
            return rows
        rows[dup] = fresh(nd)
        rows, _ = torch.sort(rows, dim=1)


def generate(cfg: InstanceConfig | str, seed: int = 0, device="cpu",
             chunk_cols: int = 1 << 23) -> Instance:
    """Build the instance of ``cfg`` (a name from CONFIGS or an InstanceConfig)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg] if cfg in CONFIGS else RAGGED_CONFIGS[cfg]
    device = torch.device(device)
    if cfg.col_lengths == "pareto":
        return _generate_ragged(cfg, seed, device)
    m, n, c = cfg.m, cfg.n, cfg.nnz_per_col
    if not (1 <= c <= m):
        raise ValueError("need 1 <= nnz_per_col <= m")
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    nnz = n * c
    rowidx = torch.empty(nnz, dtype=torch.int32, device=device)
    val = torch.empty(nnz, dtype=torch.float32, device=device)
    zcdf = _zipf_cdf(m, cfg.zipf_s, device) if cfg.rows == "zipf" else None
    for c0 in range(0, n, chunk_cols):
        k = min(chunk_cols, n - c0)
        rows = _draw_rows(k, c, m, gen, device, zcdf)
        rowidx[c0 * c:(c0 + k) * c] = rows.view(-1).to(torch.int32)
        del rows
        val[c0 * c:(c0 + k) * c] = torch.randn(k * c, generator=gen, device=device,
                                               dtype=torch.float32)
    colptr = torch.arange(0, n + 1, dtype=torch.int64, device=device) * c

    # G3: planted support
    s = min(cfg.s_star, n)
    idx = torch.empty(0, dtype=torch.int64, device=device)
    while idx.numel() < s:
        more = torch.randint(0, n, (2 * s,), generator=gen, device=device, dtype=torch.int64)
        idx = torch.unique(torch.cat([idx, more]))
    perm = torch.randperm(idx.numel(), generator=gen, device=device)[:s]
    xs_idx = torch.sort(idx[perm]).values
    xs_val = torch.randn(s, generator=gen, device=device, dtype=torch.float64)

    # G4: b = fp32(A x* + noise * eps), fp64 accumulation
    b64 = torch.zeros(m, dtype=torch.float64, device=device)
    pos = (xs_idx.view(-1, 1) * c + torch.arange(c, device=device).view(1, -1)).view(-1)
    contrib = val[pos].to(torch.float64) * xs_val.repeat_interleave(c)
    b64.index_add_(0, rowidx[pos].to(torch.int64), contrib)
    b64 += cfg.noise * torch.randn(m, generator=gen, device=device, dtype=torch.float64)
    b = b64.to(torch.float32)

    # G5: lambda = lam_frac * ||A^T b||_inf (fp64 on the fp32 b)
    bd = b.to(torch.float64)
    amax = 0.0
    for c0 in range(0, n, chunk_cols):
        k = min(chunk_cols, n - c0)
        sl = slice(c0 * c, (c0 + k) * c)
        atb = (val[sl].to(torch.float64) * bd[rowidx[sl].to(torch.int64)]).view(k, c).sum(1)
        amax = max(amax, float(atb.abs().max()))
    lam = cfg.lam_frac * amax
    return Instance(cfg, m, n, colptr, rowidx, val, b, lam, xs_idx, xs_val.to(torch.float32))


def _generate_ragged(cfg: InstanceConfig, seed: int, device) -> Instance:
    """G1-G6 with power-law column lengths (cfg.col_lengths == "pareto"): lengths
    drawn first, then each column's rows uniform and distinct (redraw duplicates),
    sorted; values N(0,1); planted x*, b and lambda as for the fixed-length configs."""
    m, n = cfg.m, cfg.n
    if cfg.len_max > m:
        raise ValueError("len_max must be <= m")
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    u = 1.0 - torch.rand(n, generator=gen, device=device, dtype=torch.float64)  # (0, 1]
    lens = torch.floor(cfg.len_min * u.pow(-1.0 / cfg.len_alpha)).clamp_(max=cfg.len_max).to(torch.int64)
    colptr = torch.zeros(n + 1, dtype=torch.int64, device=device)
    colptr[1:] = torch.cumsum(lens, 0)
    nnz = int(colptr[-1])
    col = torch.repeat_interleave(torch.arange(n, device=device), lens)
    rows = torch.randint(0, m, (nnz,), generator=gen, device=device, dtype=torch.int64)
    while True:
        key = col * m + rows
        key, _ = torch.sort(key)
        rows = key - col * m  # col is sorted, so sorting the keys keeps each column's slice
        dup = torch.zeros(nnz, dtype=torch.bool, device=device)
        dup[1:] = key[1:] == key[:-1]
        nd = int(dup.sum())
        if nd == 0:
            break
        rows[dup] = torch.randint(0, m, (nd,), generator=gen, device=device, dtype=torch.int64)
    rowidx = rows.to(torch.int32)
    del rows, key
    val = torch.randn(nnz, generator=gen, device=device, dtype=torch.float32)
    s = min(cfg.s_star, n)
    xs_idx = torch.sort(torch.randperm(n, generator=gen, device=device)[:s]).values
    xs_val = torch.randn(s, generator=gen, device=device, dtype=torch.float64)
    xfull = torch.zeros(n, dtype=torch.float64, device=device)
    xfull[xs_idx] = xs_val
    b64 = torch.zeros(m, dtype=torch.float64, device=device)
    b64.index_add_(0, rowidx.to(torch.int64), val.to(torch.float64) * xfull[col])
    b64 += cfg.noise * torch.randn(m, generator=gen, device=device, dtype=torch.float64)
    b = b64.to(torch.float32)
    atb = torch.zeros(n, dtype=torch.float64, device=device)
    atb.index_add_(0, col, val.to(torch.float64) * b.to(torch.float64)[rowidx.to(torch.int64)])
    lam = cfg.lam_frac * float(atb.abs().max())
    return Instance(cfg, m, n, colptr, rowidx, val, b, lam, xs_idx, xs_val.to(torch.float32))


def column_subset(colptr: torch.Tensor, rowidx: torch.Tensor, val: torch.Tensor, cols,
                  chunk_entries: int = 1 << 26):
    """Host CSC of the same m x n shape that keeps only the columns ``cols``
    (sorted unique int64 indices) of (colptr, rowidx, val) and leaves every other
    column empty: (colptr int64[n+1], rowidx int32, val f32) as numpy arrays.
    Pure data movement (no method arithmetic); gathers on the arrays' device in
    chunks of about ``chunk_entries`` entries so a multi-GB subset needs little
    scratch.  Used to hand the oracle the part of a large instance a run touches."""
    import numpy as np
    dev = colptr.device
    n = colptr.numel() - 1
    cols_np = np.asarray(cols, dtype=np.int64)
    ct_all = torch.from_numpy(cols_np).to(dev)
    lens_all = colptr[ct_all + 1] - colptr[ct_all]
    full = np.zeros(n + 1, dtype=np.int64)
    full[cols_np + 1] = lens_all.cpu().numpy()
    np.cumsum(full, out=full)
    total = int(full[-1])
    rows = np.empty(total, dtype=np.int32)
    vals = np.empty(total, dtype=np.float32)
    csum = torch.cumsum(lens_all, 0)
    c0, out0 = 0, 0
    while c0 < cols_np.size:
        base = int(csum[c0 - 1]) if c0 else 0
        c1 = int(torch.searchsorted(csum, base + chunk_entries, right=True))
        c1 = max(c1, c0 + 1)
        ct, lens = ct_all[c0:c1], lens_all[c0:c1]
        starts = colptr[ct]
        cnt = int(lens.sum())
        offs = torch.cumsum(lens, 0) - lens
        idx = torch.repeat_interleave(starts - offs, lens) + torch.arange(cnt, device=dev)
        rows[out0:out0 + cnt] = rowidx[idx].cpu().numpy()
        vals[out0:out0 + cnt] = val[idx].cpu().numpy()
        out0 += cnt
        c0 = c1
        del idx, starts, offs
    assert out0 == total
    return full, rows, vals


def random_csc(m: int, n: int, col_lengths, seed: int = 0, device="cpu",
               values: str = "normal"):
    """Small ragged CSC for edge-case tests: column i gets col_lengths[i]
    distinct uniform rows (sorted).  Returns (colptr int64, rowidx int32, val f32)."""
    gen = torch.Generator(device="cpu")
    gen.manual_seed(seed)
    lens = [int(v) for v in col_lengths]
    rows, vals = [], []
    for ln in lens:
        if ln > m:
            raise ValueError("column longer than m")
        r = torch.randperm(m, generator=gen)[:ln].sort().values
        rows.append(r)
        if values == "normal":
            vals.append(torch.randn(ln, generator=gen, dtype=torch.float32))
        else:
            vals.append(torch.ones(ln, dtype=torch.float32))
    colptr = torch.zeros(n + 1, dtype=torch.int64)
    colptr[1:] = torch.cumsum(torch.tensor(lens, dtype=torch.int64), 0)
    rowidx = torch.cat(rows).to(torch.int32) if rows else torch.zeros(0, dtype=torch.int32)
    val = torch.cat(vals) if vals else torch.zeros(0, dtype=torch.float32)
    return colptr.to(device), rowidx.to(device), val.to(device)


def random_b(m: int, seed: int = 0, device="cpu") -> torch.Tensor:
    gen = torch.Generator(device="cpu")
    gen.manual_seed(seed + 7919)
    return torch.randn(m, generator=gen, dtype=torch.float32).to(device)


def lam_for(colptr, rowidx, val, b, frac: float = 0.1) -> float:
    """G5 on an arbitrary small CSC (host tensors)."""
    n = colptr.numel() - 1
    col = torch.repeat_interleave(torch.arange(n), (colptr[1:] - colptr[:-1]))
    atb = torch.zeros(n, dtype=torch.float64)
    atb.index_add_(0, col, val.double() * b.double()[rowidx.long()])
    return frac * float(atb.abs().max()) if n else 0.0


def equal_row_01_matrix(m: int, n: int, omega: int, seed: int = 0):
    """0-1 matrix with exactly ``omega`` ones per row and k = omega*m/n ones per
    column (the DSO tightness construction).  Rows are
    consecutive cyclic windows of a random column permutation; requires
    omega*m % n == 0.  Returns a host CSC (colptr, rowidx, val)."""
    if (omega * m) % n:
        raise ValueError("need omega*m divisible by n")
    gen = torch.Generator(device="cpu")
    gen.manual_seed(seed)
    perm = torch.randperm(n, generator=gen)
    cols = [[] for _ in range(n)]
    for j in range(m):
        for t in range(omega):
            cols[int(perm[(j * omega + t) % n])].append(j)
    lens = [len(cl) for cl in cols]
    colptr = torch.zeros(n + 1, dtype=torch.int64)
    colptr[1:] = torch.cumsum(torch.tensor(lens), 0)
    rowidx = torch.tensor([r for cl in cols for r in sorted(cl)], dtype=torch.int32)
    val = torch.ones(rowidx.numel(), dtype=torch.float32)
    return colptr, rowidx, val


def equal_row_random_matrix(m: int, n: int, omega: int, seed: int = 0):
    """0-1 matrix with exactly ``omega`` ones per row and k = omega*m/n ones per
    column, rows drawn at random (the Sec. 8.2 "theory versus reality" matrices,
    PAPER.md:1289, built on the DSO tightness construction PAPER.md:697-703):
    rows come in k blocks of n/omega; block t splits a fresh random permutation
    of the columns into n/omega groups of omega.  Needs n % omega == 0 and
    m % (n/omega) == 0.  Returns a host CSC (colptr, rowidx, val)."""
    if n % omega or m % (n // omega):
        raise ValueError("need omega | n and (n/omega) | m")
    g = n // omega
    gen = torch.Generator(device="cpu")
    gen.manual_seed(seed)
    cols_of_row = []
    for t in range(m // g):
        perm = torch.randperm(n, generator=gen).view(g, omega)
        cols_of_row.append(perm)
    rows_cols = torch.cat(cols_of_row, 0)                      # [m, omega]
    row_ids = torch.arange(m).repeat_interleave(omega)
    col_ids = rows_cols.reshape(-1)
    order = torch.argsort(col_ids * m + row_ids)
    col_sorted, row_sorted = col_ids[order], row_ids[order]
    counts = torch.bincount(col_sorted, minlength=n)
    colptr = torch.zeros(n + 1, dtype=torch.int64)
    colptr[1:] = torch.cumsum(counts, 0)
    return colptr, row_sorted.to(torch.int32), torch.ones(m * omega, dtype=torch.float32)


# L2-regularised logistic regression (Sec. 8.4): KDDB is not
# available, so a synthetic instance with its shape stands in for it (DESIGN.md
# "Input recipe"): n features (columns), m examples (rows), c nonzeros per feature
# at uniform distinct examples, N(0,1) values, labels y = sign(A w* + 0.1 eps) with
# a 1 %-dense planted w*, lambda = 1 (the paper's value).
LOGISTIC_CONFIGS = {
    "logistic_small": InstanceConfig("logistic_small", 20_000, 30_000, 19, 300, tau=1024, iters=2000),
    "kddb_like": InstanceConfig("kddb_like", 19_264_097, 29_890_095, 19, 298_900, tau=1 << 16, iters=500),
}


def generate_logistic(cfg, seed: int = 0, device="cpu", lam: float = 1.0, chunk_cols: int = 1 << 23):
    """(colptr, rowidx, val, y, lam) for a logistic config (name or InstanceConfig)."""
    if isinstance(cfg, str):
        cfg = LOGISTIC_CONFIGS[cfg]
    device = torch.device(device)
    m, n, c = cfg.m, cfg.n, cfg.nnz_per_col
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    rowidx = torch.empty(n * c, dtype=torch.int32, device=device)
    val = torch.empty(n * c, dtype=torch.float32, device=device)
    for c0 in range(0, n, chunk_cols):
        k = min(chunk_cols, n - c0)
        rows = _draw_rows(k, c, m, gen, device, None)
        rowidx[c0 * c:(c0 + k) * c] = rows.view(-1).to(torch.int32)
        del rows
        val[c0 * c:(c0 + k) * c] = torch.randn(k * c, generator=gen, device=device, dtype=torch.float32)
    colptr = torch.arange(0, n + 1, dtype=torch.int64, device=device) * c
    s = min(cfg.s_star, n)
    widx = torch.randperm(n, generator=gen, device=device)[:s]
    wval = torch.randn(s, generator=gen, device=device, dtype=torch.float64)
    z = torch.zeros(m, dtype=torch.float64, device=device)
    pos = (widx.view(-1, 1) * c + torch.arange(c, device=device).view(1, -1)).view(-1)
    z.index_add_(0, rowidx[pos].to(torch.int64), val[pos].to(torch.float64) * wval.repeat_interleave(c))
    z += 0.1 * torch.randn(m, generator=gen, device=device, dtype=torch.float64)
    y = torch.where(z >= 0, 1.0, -1.0).to(torch.float32)
    return colptr, rowidx, val, y, float(lam)
