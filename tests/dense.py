"""Independent dense / scalar oracles (tests/oracles.hpp:14-143 restated in
numpy): straight-line residual with an explicit cos/sin rotation matrix,
central finite differences, dense reconstructions of B, C, E and the Schur
operator."""
import numpy as np


def residual_reference(cam, pt, pix):
    """tests/oracles.hpp:20-47."""
    aa = np.asarray(cam[:3], float)
    th = np.linalg.norm(aa)
    if th < 1e-14:
        R = np.eye(3) + np.array([[0, -aa[2], aa[1]], [aa[2], 0, -aa[0]], [-aa[1], aa[0], 0]])
    else:
        a = aa / th
        K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
        R = np.cos(th) * np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * np.outer(a, a)
    p = R @ np.asarray(pt, float) + np.asarray(cam[3:6], float)
    u = -p[:2] / p[2]
    n2 = u @ u
    d = 1 + cam[7] * n2 + cam[8] * n2 * n2
    return cam[6] * d * u - np.asarray(pix, float)


def fd_jacobian(resid, cam, pt, pix):
    """Central differences, h = 1e-7 max(1, |p|) (tests/oracles.hpp:51-82)."""
    params = np.concatenate([cam, pt]).astype(float)
    J = np.zeros((2, 12))
    for j in range(12):
        h = 1e-7 * max(1.0, abs(params[j]))
        hi, lo = params.copy(), params.copy()
        hi[j] += h
        lo[j] -= h
        J[:, j] = (resid(hi[:9], hi[9:], pix) - resid(lo[:9], lo[9:], pix)) / (2 * h)
    return J


def dense_blockdiag(blocks):
    blocks = np.asarray(blocks, float)
    nb, bs = blocks.shape[0], blocks.shape[1]
    out = np.zeros((nb * bs, nb * bs))
    for i in range(nb):
        out[i * bs:(i + 1) * bs, i * bs:(i + 1) * bs] = blocks[i]
    return out


def dense_coupling(E, cam_ids, pt_ids, m, n):
    out = np.zeros((9 * m, 3 * n))
    for e, (c, p) in enumerate(zip(cam_ids, pt_ids)):
        out[9 * c:9 * c + 9, 3 * p:3 * p + 3] += E[e]
    return out


def dense_jacobian(jac, res, cam_ids, pt_ids, w, m, n):
    """Scatter of the per-edge blocks (tests/oracles.hpp:85-114); jac (2,12,N)."""
    N = len(cam_ids)
    J = np.zeros((2 * N, 9 * m + 3 * n))
    r = np.zeros(2 * N)
    for e in range(N):
        s = np.sqrt(w[e])
        J[2 * e:2 * e + 2, 9 * cam_ids[e]:9 * cam_ids[e] + 9] = s * jac[:, :9, e]
        J[2 * e:2 * e + 2, 9 * m + 3 * pt_ids[e]:9 * m + 3 * pt_ids[e] + 3] = s * jac[:, 9:, e]
        r[2 * e:2 * e + 2] = s * res[:, e]
    return J, r


def damp_dense(D, lam, policy):
    D = D.copy()
    d = np.diag(D).copy()
    if policy == 0:
        D[np.diag_indices_from(D)] = d + lam
    else:
        D[np.diag_indices_from(D)] = d + lam * np.clip(d, 1e-6, 1e32)
    return D


def schur(Bd, Cd, E):
    return Bd - E @ np.linalg.solve(Cd, E.T)


def rel(a, b, floor=1.0):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(floor, np.linalg.norm(b)))
