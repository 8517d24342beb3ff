"""Algorithmic flop / byte model of the build (frozen before tuning).

Minimal-work counts: FMA = 2 flops, complex x real = 2, complex x complex = 6 + 2; zero structure of
the cross-product maps not counted; transcendentals counted as 1.  Per (target, patch) pair, all four
kernels S, D, S', D':
  F_tgt  = 12 (p+3)^2                                   target harmonics (Step 4)
  F_Q    = 36 * 3p~ * n_Q, F_dQ = F_Q, F_V = 12 * 3p~ * n_V   line-integral maps (Step 6)
  F_tr   = 20 T_lam + 40 T_lam + 4 T_theta              translation (Step 7)
  F_edge = 3 (6 p~^2 + 300 p~) + 2 n_Omega (12 p~ + 40) per swap-regime edge   (Step 5)
  F_con  = 8 n_p n (D) + 8 n_p n (D') + 10 n_p n (S) + 8 n_p n + 40 n_p (S')   (Step 8)
Per kernel: k_pair_edge F_tgt + F_edge (+ swap extras); k_qmap F_Q + F_dQ + F_V; k_translate F_tr;
k_contract F_con.  A kernel mask counts only the selected kernels' work (the build skips the rest): F_dQ and
the 40 T_lam dW terms with D', F_V and the 4 T_theta terms with S, each kernel's own contraction; F_Q and the
20 T_lam W terms with any kernel.
Algorithmic bytes per pair: the CSR output (4 n fp64 values + n int32 columns) + target (56 B); the
patch data is amortised over the pairs of a patch (added per patch).
"""


def translation_terms(p, jmin):
    n = 0
    for l in range(1, p + 1):
        for m in range(1, l + 1):
            for j in range(jmin, l + 1):
                for k in range(-j, j + 1):
                    if abs(m - k) <= l - j:
                        n += 1
    return n


def pair_flops(p, q=None, n_omega=32, mask=15):
    q = q or 2 * p
    n, npb = p * p, p * (p + 1) // 2
    ns = (p + 1) * (p + 2) // 2
    nq, nv = ns - 3, ns - 1
    tl, tt = translation_terms(p, 2), translation_terms(p, 1)
    S, D, Sp, Dp = (mask >> 0) & 1, (mask >> 1) & 1, (mask >> 2) & 1, (mask >> 3) & 1
    edge = 12 * (p + 3) ** 2 + 3 * (6 * q * q + 300 * q)
    qmap = (1 + Dp) * 36 * 3 * q * nq + S * 12 * 3 * q * nv
    translate = 20 * tl + Dp * 40 * tl + S * 4 * tt
    zeta = edge + qmap + translate
    contract = 8 * npb * n * (D + Dp) + S * 10 * npb * n + Sp * (8 * npb * n + 40 * npb)
    swap_edge = 2 * n_omega * (12 * q + 40)
    return dict(edge=edge, qmap=qmap, translate=translate, zeta=zeta, contract=contract, swap_edge=swap_edge,
                total=zeta + contract)


def pair_bytes(p):
    n = p * p
    return 4 * n * 8 + n * 4 + 56


if __name__ == "__main__":
    for p in (4, 6, 8, 10):
        print(p, pair_flops(p))
