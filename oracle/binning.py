"""Block partition of the nodes (TEST INFRASTRUCTURE ONLY).

PAPER.md:520-527 splits the torus into equally sized blocks R_p and collects
Gamma_p = {j : k_j in R_p}; PAPER.md:533 partitions I_Ntilde into blocks of
Q = ceil(Ntilde / P) cells. The normative integer form (reading R10)
bins every node by the grid cell its footprint starts from:

    t_d = Ntilde_d * k_d        (one IEEE fp64 multiplication; k promoted to fp64)
    a_d = floor(t_d)
    c_d = (a_d + Ntilde_d/2) mod Ntilde_d     (cell of [-1/2,1/2)-centred grid)
    p_d = floor(c_d / Q_d),  P_d = ceil(Ntilde_d / Q_d)
    key = C-order linear index of p (last dimension fastest)

perm lists node indices grouped by key ascending, ties by original index
(stable, reading R12); offsets[p] is the start of tile p in perm
(length prod(P) + 1).
"""

import numpy as np


def tile_keys(nodes, Ntilde, Q):
    nodes = np.asarray(nodes).reshape(-1, len(Ntilde)).astype(np.float64)
    key = np.zeros(nodes.shape[0], dtype=np.int64)
    P = []
    for d, (nt, q) in enumerate(zip(Ntilde, Q)):
        t = float(nt) * nodes[:, d]
        a = np.floor(t).astype(np.int64)
        c = np.mod(a + nt // 2, nt)
        p = c // q
        Pd = -(-nt // q)
        P.append(Pd)
        key = key * Pd + p
    return key, tuple(P)


def bin_nodes(nodes, Ntilde, Q):
    """Returns (perm int64[M], offsets int64[prod(P)+1], P)."""
    key, P = tile_keys(nodes, Ntilde, Q)
    perm = np.argsort(key, kind="stable")
    counts = np.bincount(key, minlength=int(np.prod(P)))
    offsets = np.concatenate([[0], np.cumsum(counts)])
    return perm, offsets, P
