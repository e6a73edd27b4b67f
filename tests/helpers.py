"""Test-side helpers: layout packing only (no DCNv4 arithmetic)."""
import numpy as np

import oracle


def pack_om(dx, dy, m, S=None):
    """Fused offset_mask row [N,Ho,Wo,S] from dx, dy, m of shape [N,Ho,Wo,G,K].

    Layout (reading R3): group g occupies channels g*3K .. g*3K+3K-1 as
    [dx_0, dy_0, dx_1, dy_1, ..., dx_{K-1}, dy_{K-1}, m_0, ..., m_{K-1}]."""
    N, Ho, Wo, G, K = m.shape
    S = S or 3 * G * K
    om = np.zeros((N, Ho, Wo, S), np.float64)
    body = om[..., : 3 * G * K].reshape(N, Ho, Wo, G, 3 * K)
    body[..., 0: 2 * K: 2] = dx
    body[..., 1: 2 * K: 2] = dy
    body[..., 2 * K:] = m
    om[..., : 3 * G * K] = body.reshape(N, Ho, Wo, 3 * G * K)
    return om


def unpack_om(om, G, K):
    """Inverse of pack_om: (dx, dy, m) each [N,Ho,Wo,G,K]."""
    N, Ho, Wo, S = om.shape
    body = np.asarray(om)[..., : 3 * G * K].reshape(N, Ho, Wo, G, 3 * K)
    return body[..., 0: 2 * K: 2], body[..., 1: 2 * K: 2], body[..., 2 * K:]


def geom(**kw):
    return oracle.Geometry(**kw)


def rng_case(seed, g: oracle.Geometry, off_lo=-2.0, off_hi=2.0):
    rs = np.random.RandomState(seed)
    Ho, Wo = g.out_hw()
    x = rs.uniform(-1, 1, (g.N, g.H, g.W, g.C))
    dx = rs.uniform(off_lo, off_hi, (g.N, Ho, Wo, g.G, g.K))
    dy = rs.uniform(off_lo, off_hi, (g.N, Ho, Wo, g.G, g.K))
    m = rs.uniform(-1, 1, (g.N, Ho, Wo, g.G, g.K))
    gy = rs.uniform(-1, 1, (g.N, Ho, Wo, g.C))
    return x, pack_om(dx, dy, m, g.S), gy
