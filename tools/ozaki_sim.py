"""Host simulation of the exact integer-sliced recurrent update (design check).

x = U[w] + W h is computed from 8-bit digit planes of W (per output row scale,
top plane signed, lower planes unsigned) and of h (per context row scale, all
planes unsigned), 13 plane pairs (a + b <= 4) accumulated exactly in int32
per anti-diagonal s = a + b, then combined in float64.  The f32 rounding of
sigmoid(x) is certified against a rigorous bound on |x~ - x_ref|; uncertain
elements fall back to the reference's sequential float64 sum.  Reports how
often the fallback is needed and checks the certified values against the C
oracle's bit-exact advance_hidden.
"""
import sys
import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402


def w_planes(W):
    H = W.shape[1]
    mx = np.abs(W).max(axis=1)
    e = np.where(mx > 0, np.floor(np.log2(np.where(mx > 0, mx, 1))) + 1, 0).astype(np.int64)
    sW = np.ldexp(1.0, e)                                  # |W| / sW < 1
    X = np.rint(W.astype(np.float64) / sW[:, None] * 2.0 ** 31).astype(np.int64)
    d0 = X >> 24
    R = X - (d0 << 24)
    planes = [d0, (R >> 16) & 255, (R >> 8) & 255, R & 255]
    err = np.abs(X * 2.0 ** -31 * sW[:, None] - W.astype(np.float64)).sum(axis=1)   # sum |dW| per row
    return planes, sW, err


def h_planes(h):
    mx = h.max(axis=1)
    e = (np.floor(np.log2(mx)) + 1).astype(np.int64)
    sH = np.ldexp(1.0, e)
    Y = np.rint(h.astype(np.float64) / sH[:, None] * 2.0 ** 32).astype(np.int64)
    assert Y.max() < 2 ** 32
    planes = [(Y >> 24) & 255, (Y >> 16) & 255, (Y >> 8) & 255, Y & 255]
    err = np.abs(Y * 2.0 ** -32 * sH[:, None] - h.astype(np.float64)).max(axis=1)   # max |dh| per row
    return planes, sH, err


def main(H=256, n=2000, seed=0):
    rng = np.random.default_rng(seed)
    W = rng.uniform(-0.1, 0.1, (H, H)).astype(np.float32)
    U = rng.uniform(-0.1, 0.1, (n, H)).astype(np.float32)
    h = (1 / (1 + np.exp(-rng.normal(0, 1, (n, H))))).astype(np.float32)
    wp, sW, eW = w_planes(W)
    hp, sH, eH = h_planes(h)
    # diagonals
    D = [np.zeros((H, n), np.int64) for _ in range(5)]
    for a in range(4):
        for b in range(4):
            if a + b <= 4:
                D[a + b] += wp[a] @ hp[b].T
    assert max(np.abs(d).max() for d in D) < 2 ** 31
    S = sum(D[s].astype(np.float64) * 2.0 ** (-8 * s) for s in range(5)) * 2.0 ** -15
    x = U.T.astype(np.float64) + S * sW[:, None] * sH[None, :]
    # rigorous bound: dropped pairs + representation + reference rounding
    sumW = np.abs(W.astype(np.float64)).sum(axis=1)
    drop = np.zeros(H)
    for a in range(4):
        for b in range(4):
            if a + b > 4:
                drop_ab = np.abs(wp[a]).sum(axis=1) * 255.0
                drop += drop_ab * 2.0 ** (-15 - 8 * (a + b))
    eps = drop[:, None] * sW[:, None] * sH[None, :] + eW[:, None] * 1.0 + sumW[:, None] * eH[None, :]
    eps += 600 * 2.0 ** -53 * (np.abs(U.T) + sumW[:, None])
    sig = 1 / (1 + np.exp(-x))
    y = sig.astype(np.float32)
    # midpoints around y
    yu = y.view(np.uint32)
    up = (yu + 1).view(np.float32).astype(np.float64)
    dn = (yu - 1).view(np.float32).astype(np.float64)
    m_hi = (y.astype(np.float64) + up) / 2
    m_lo = (y.astype(np.float64) + dn) / 2
    z = 1 + np.exp(-x)
    dz = eps * 1.0 + 4e-16
    cert = (z * m_lo - 1 < -dz) & (z * m_hi - 1 > dz)
    ref = np.stack([O.advance_hidden(U[r], W, h[r]) for r in range(n)], axis=1)
    ok = y == ref
    print(f"H={H}: max eps {eps.max():.3e}, certified {cert.mean()*100:.3f}%, "
          f"certified-but-wrong {(cert & ~ok).sum()}, uncertified {(~cert).sum()} of {cert.size}, "
          f"plain-round mismatches {(~ok).sum()}")


if __name__ == "__main__":
    for H in (256, 512):
        main(H, 1000 if H == 512 else 2000)
