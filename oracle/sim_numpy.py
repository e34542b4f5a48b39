"""Independent numpy restatement of simulate(steps) -- TEST INFRASTRUCTURE ONLY.

Parity unpinned against the reference (it has no spike loop; see
oracle/sim_oracle.c).  This second restatement exists to pin the C oracle:
both are written from DESIGN.md section 3 with different data structures
(dense float32 vector ops and an explicit synapse list here, a CSR loop there)
and must agree bit for bit.  Small networks only (pure numpy, O(steps * S)).
"""

from __future__ import annotations

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
TAG_DRIVE = 0xD21E0001
TAG_VINIT = 0x1417AB01
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, seed: int):
    """Vectorised Philox4x32-10 over uint32 arrays; returns four uint32 arrays."""
    c = [np.asarray(x, dtype=np.uint32).copy() for x in (c0, c1, c2, c3)]
    c = np.broadcast_arrays(*c)
    c = [x.astype(np.uint32) for x in c]
    k0 = np.uint32(seed & 0xFFFFFFFF)
    k1 = np.uint32((seed >> 32) & 0xFFFFFFFF)
    for _ in range(10):
        p0 = M0 * c[0].astype(np.uint64)
        p1 = M1 * c[2].astype(np.uint64)
        hi0 = (p0 >> np.uint64(32)).astype(np.uint32)
        lo0 = (p0 & MASK32).astype(np.uint32)
        hi1 = (p1 >> np.uint64(32)).astype(np.uint32)
        lo1 = (p1 & MASK32).astype(np.uint32)
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
        k0 = np.uint32((int(k0) + int(W0)) & 0xFFFFFFFF)
        k1 = np.uint32((int(k1) + int(W1)) & 0xFFFFFFFF)
    return c


def simulate_numpy(n, edges_i, edges_j, q_edge, owner, n_shards, next_hop, lif: dict, steps: int):
    """Return (raster[steps, n] bool, deliv[steps, S, S], hop[steps, S, S], v, i).

    ``lif`` holds the fp32-ready constants (the same dict the C oracle gets).
    Synapses: each undirected edge (i, j, q) drives j from i and i from j.
    """
    f32 = np.float32
    gid = np.arange(n, dtype=np.uint32)
    seed = int(lif["seed"])
    # synapse list (pre -> post) and signed integer weights
    pre = np.concatenate([edges_i, edges_j]).astype(np.int64)
    post = np.concatenate([edges_j, edges_i]).astype(np.int64)
    qq = np.concatenate([q_edge, q_edge]).astype(np.int64)
    every = int(lif["inh_every"])
    inh = (pre % every == every - 1) if every > 0 else np.zeros(pre.size, dtype=bool)
    wint = np.where(inh, -int(lif["g_inh"]) * qq, qq)

    r = philox4x32_10(gid, np.uint32(0xFFFFFFFF), np.uint32(TAG_VINIT), np.uint32(0), seed)
    u = (r[0] >> np.uint32(8)).astype(f32) * f32(5.9604644775390625e-08)
    v = (f32(lif["v_reset"]) + u * f32(lif["v_init_span"])).astype(f32)
    isyn = np.zeros(n, dtype=f32)
    ref = np.zeros(n, dtype=np.int32)
    fired_prev = np.zeros(n, dtype=bool)

    owner = np.asarray(owner, dtype=np.int64)
    S = int(n_shards)
    nh = np.asarray(next_hop, dtype=np.int64).reshape(S, S)
    dest = np.zeros((n, S), dtype=bool)
    dest[pre, owner[post]] = True          # pre drives post, so post's shard hosts a target of pre
    dest[np.arange(n), owner] = False

    raster = np.zeros((steps, n), dtype=bool)
    deliv = np.zeros((steps, S, S), dtype=np.int64)
    hop = np.zeros((steps, S, S), dtype=np.int64)
    thr = np.uint32(lif["ext_threshold"])
    lanes = int(lif["ext_lanes"])
    for t in range(steps):
        acc = np.zeros(n, dtype=np.int64)
        np.add.at(acc, post, np.where(fired_prev[pre], wint, 0))
        acc = acc.astype(np.int32)
        if lanes > 0:
            rr = philox4x32_10(gid, np.uint32(t), np.uint32(TAG_DRIVE), np.uint32(0), seed)
            ext = sum((rr[k] < thr).astype(np.int32) for k in range(min(lanes, 4)))
        else:
            ext = np.zeros(n, dtype=np.int32)
        syn = acc.astype(f32)
        isyn = (isyn * f32(lif["alpha_i"]) + syn * f32(lif["w_unit"])).astype(f32)
        isyn = (isyn + ext.astype(f32) * f32(lif["w_ext"])).astype(f32)
        refr = ref > 0
        vn = (f32(lif["v_rest"]) + (v - f32(lif["v_rest"])) * f32(lif["alpha_v"])).astype(f32)
        vn = (vn + isyn * f32(lif["beta"])).astype(f32)
        fired = (~refr) & (vn >= f32(lif["v_th"]))
        v = np.where(refr | fired, f32(lif["v_reset"]), vn).astype(f32)
        ref = np.where(refr, ref - 1, np.where(fired, int(lif["t_ref"]), ref))
        raster[t] = fired
        for i in np.flatnonzero(fired & dest.any(axis=1)).tolist():
            s = owner[i]
            ds = np.flatnonzero(dest[i])
            deliv[t, s, ds] += 1
            hops = nh[s, ds]
            if (hops < 0).any():
                raise ValueError("destination without a next hop")
            for h in np.unique(hops).tolist():
                hop[t, s, h] += 1
                behind = ds[(hops == h) & (ds != h)]
                hop[t, h, behind] += 1
        fired_prev = fired
    return raster, deliv, hop, v, isyn
