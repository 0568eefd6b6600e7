"""HBM weight layouts of the cfb kernels (torch, on device; see include/cfb.h).

Row tiles (csrc/gemv.cuh): rows grouped 4 at a time and stored chunk-major,
[tile][16-byte chunk][4 rows][chunk elements], so a warp's weight load is 512
contiguous bytes and the streaming unit is a contiguous byte range.
"""

from __future__ import annotations

TILE_ROWS = 4


def _epc(t) -> int:
    """elements per 16-byte chunk"""
    return 16 // t.element_size()


def row_tiles(w, rows_pad: int | None = None):
    """(..., R, C) -> (..., R_pad/4, C/epc, 4, epc), zero rows appended."""
    import torch
    *lead, R, C = w.shape
    rp = rows_pad if rows_pad is not None else -(-R // TILE_ROWS) * TILE_ROWS
    if rp != R:
        pad = torch.zeros(*lead, rp - R, C, device=w.device, dtype=w.dtype)
        w = torch.cat([w, pad], dim=-2)
    e = _epc(w)
    return w.reshape(*lead, rp // TILE_ROWS, TILE_ROWS, C // e, e).transpose(-3, -2).contiguous()


def gate_up_tiles(w1, w2):
    """w1, w2 (F, D) -> tiles of rows (w1[2t], w1[2t+1], w2[2t], w2[2t+1])."""
    import torch
    F, D = w1.shape
    inter = torch.cat([w1.reshape(F // 2, 2, D), w2.reshape(F // 2, 2, D)], dim=1)  # (F/2, 4, D)
    e = _epc(w1)
    return inter.reshape(F // 2, TILE_ROWS, D // e, e).transpose(1, 2).contiguous()


def qkv_tiles(w_qkv, n_blocks: int, head_pad: int, hidden_pad: int):
    """(nh, D, 3H) -> [nh][N][tiles of rows (q slice | k slice | v slice) of
    head_pad/N dims each][D']: rank r's rows are q[r*h:(r+1)*h], k[...], v[...]."""
    import torch
    nh, D, threeH = w_qkv.shape
    H = threeH // 3
    hp = head_pad // n_blocks
    w = w_qkv.reshape(nh, D, 3, H).permute(0, 2, 3, 1)  # (nh, 3, H, D)
    wp = torch.zeros(nh, 3, head_pad, hidden_pad, device=w.device, dtype=w.dtype)
    wp[:, :, :H, :D] = w
    rows = wp.reshape(nh, 3, n_blocks, hp, hidden_pad).permute(0, 2, 1, 3, 4)  # (nh, N, 3, h, D')
    rows = rows.reshape(nh, n_blocks, 3 * hp, hidden_pad)
    return row_tiles(rows)


def wo_rows(w_out_t, n_blocks: int):
    """(nh, D, Hp) = (W_out[head])^T -> [nh][N][D/N][Hp]: rank r's rows
    r*D/N .. (r+1)*D/N, each row chunk-rotated for the row-per-lane O-proj
    (csrc/gemv.cuh rowlane_item): logical 16-byte chunk k of slice row g is
    stored at chunk (k + g) mod nch."""
    import torch
    nh, D, Hp = w_out_t.shape
    cols = D // n_blocks
    e = _epc(w_out_t)
    nch = Hp // e
    w = w_out_t.reshape(nh, n_blocks, cols, nch, e)
    g = torch.arange(cols, device=w.device).view(cols, 1)
    p = torch.arange(nch, device=w.device).view(1, nch)
    logical = (p - g) % nch  # physical chunk p holds logical chunk (p - g) mod nch
    idx = logical.view(1, 1, cols, nch, 1).expand(nh, n_blocks, cols, nch, e)
    return torch.gather(w, 3, idx).reshape(nh, n_blocks, cols, Hp).contiguous()


def rotated_rows(t):
    """(..., rows, C) -> same shape with every row chunk-rotated by its index
    g within the rows dim: logical 16-byte chunk k stored at (k + g) mod nch
    (the row-per-lane GEMV layout, csrc/gemv.cuh rowlane_item)."""
    import torch
    *lead, rows, C = t.shape
    e = _epc(t)
    nch = C // e
    w = t.reshape(*lead, rows, nch, e)
    g = torch.arange(rows, device=t.device).view(rows, 1)
    p = torch.arange(nch, device=t.device).view(1, nch)
    logical = ((p - g) % nch).view(*([1] * len(lead)), rows, nch, 1).expand(*lead, rows, nch, e)
    return torch.gather(w, len(lead) + 1, logical).reshape(*lead, rows, C).contiguous()

