"""Algorithmic cost model of the BASELINE configs.

Two figures per unit of work, both independent of how the kernels are written:

* B_alg  compulsory HBM bytes: every input ciphertext / plaintext / key read once,
         every output ciphertext written once (8-byte words);
* M_alg  modular multiplications of the op sequence, with one NTT of one limb
         = (N/2) log2 N butterflies (one modmul each).

Formulas (l = limbs at the operating level, N = ring degree), SURVEY.md 8(d):
    ct = 2 l N words; key = 2 l (l+1) N words (dnum = l digits, one special prime)
    tensor = 4 l N;  ks(l) = (l+1)(l+2) ntt + 2 l (l+1) N + 4 l N
    rescale(l) = 2 l ntt + 2 (l-1) N;  pt x ct (or scalar x ct) = 2 l N
    mul(l) = tensor + ks + rescale;  act(l) = mul(l) + 2 pt x ct (c3 = 0: x^2, c1 x, c2 x^2)
bench.py turns them into roofline fractions: t_min = max(B_alg / HBM peak, M_alg / P_modmul),
frac = t_min / t_measured; the per-resource fractions are reported beside it.
"""

from __future__ import annotations

import math

W = 8  # bytes per residue word


def ntt(N: int) -> float:
    return N / 2 * math.log2(N)


def ct_bytes(l: int, N: int) -> float:
    return 2 * l * N * W


def pt_bytes(l: int, N: int) -> float:
    return l * N * W


def key_bytes(l: int, N: int) -> float:
    return 2 * l * (l + 1) * N * W


def tensor(l: int, N: int) -> float:
    return 4 * l * N


def ks(l: int, N: int) -> float:
    return (l + 1) * (l + 2) * ntt(N) + 2 * l * (l + 1) * N + 4 * l * N


def rescale(l: int, N: int) -> float:
    return 2 * l * ntt(N) + 2 * (l - 1) * N


def ptct(l: int, N: int) -> float:
    return 2 * l * N


def mul(l: int, N: int) -> float:
    return tensor(l, N) + ks(l, N) + rescale(l, N)


def act(l: int, N: int) -> float:
    return mul(l, N) + 2 * ptct(l, N)


def matmul(n: int, nb: int, l: int, N: int) -> tuple[float, float]:
    """matmul_outer over n column-ciphertext pairs, nb row blocks sharing R (fused: one relin +
    rescale per block).  Per HE matmul."""
    B = (nb * n + n) * ct_bytes(l, N) + key_bytes(l, N) + nb * ct_bytes(l - 1, N)
    M = nb * (n * tensor(l, N) + ks(l, N) + rescale(l, N))
    return B, M


def conv_act(C: int, W_in: int, k: int, F: int, out_cols: int, l: int, N: int, activation: bool = True):
    """One conv layer (+ degree-2 activation) on column ciphertexts: C channels x W_in input
    columns at l limbs, F filters, out_cols output columns.  Per batch (one ciphertext set)."""
    rots = C * W_in * (k - 1)  # rotated copies, one key switch each (the reference caches per call)
    outs = F * out_cols
    B = C * W_in * ct_bytes(l, N) + key_bytes(l, N) * (k - 1 + (1 if activation else 0))
    M = rots * ks(l, N) + outs * C * k * k * ptct(l, N) + outs * rescale(l, N)
    if activation:
        B += outs * ct_bytes(l - 3, N)
        M += outs * act(l - 1, N)
    else:
        B += outs * ct_bytes(l - 1, N)
    return B, M


def cfg3(N: int = 1 << 14, L: int = 5, m: int = 64, h: int = 28, F: int = 5, k: int = 4, ny: int = 64, nz: int = 10):
    """Config 3 per pass of m images: stride-2 conv (13 output columns) -> square -> dense
    845 -> 64 (F*13 plaintext products per neuron, 5 in-block rotations) -> square -> dense 64 -> 10."""
    l0 = L + 1
    no = len(range(0, h - k + 1, 2))
    B, M = conv_act(1, h, k, F, no, l0, N, activation=False)  # conv at l0 -> l0-1
    feats = F * no
    l1 = l0 - 1
    M += feats * mul(l1, N)  # square -> l1-1
    l2 = l1 - 1
    B += ny * feats * pt_bytes(l2, N) + key_bytes(l1, N)  # dense-1 plaintexts, relin key
    M += ny * feats * ptct(l2, N) + ny * rescale(l2, N)
    l3 = l2 - 1
    B += 3 * key_bytes(l3, N)  # block-sum Galois keys
    M += ny * 5 * ks(l3, N)
    M += ny * mul(l3, N)  # square
    l4 = l3 - 1
    B += nz * ny * pt_bytes(l4, N)
    M += nz * ny * ptct(l4, N) + nz * rescale(l4, N)
    B += nz * ct_bytes(l4 - 1, N)
    return B, M


def cfg4(N: int = 1 << 15, L: int = 7, C: int = 3, W_in: int = 226, k: int = 3, F: int = 16, out_cols: int = 224):
    """Config 4 per batch (one set of column ciphertexts: 16 images at cfg 4, 64 at cfg 5b)."""
    return conv_act(C, W_in, k, F, out_cols, L + 1, N, activation=True)


CONFIGS = {
    1: lambda: matmul(8, 1, 2, 1 << 13),
    2: lambda: matmul(64, 1, 5, 1 << 14),
    "5a": lambda: matmul(256, 4, 8, 1 << 15),
    3: cfg3,
    4: cfg4,
    "5b": cfg4,
}


def roofline(B: float, M: float, t: float, hbm_gbs: float, modmul_gs: float) -> dict:
    """Roofline fractions of one unit of work measured at t seconds."""
    t_hbm = B / (hbm_gbs * 1e9)
    t_int = M / (modmul_gs * 1e9)
    t_min = max(t_hbm, t_int)
    return {"bound": "hbm" if t_hbm >= t_int else "int", "frac": t_min / t, "t_min_us": t_min * 1e6, "t_us": t * 1e6,
            "B_alg_bytes": B, "M_alg_modmul": M, "hbm_frac": (B / t) / (hbm_gbs * 1e9),
            "int_frac": (M / t) / (modmul_gs * 1e9), "peak_hbm_gbs": hbm_gbs, "peak_modmul_gs": modmul_gs}
