"""Test problem factories (tests/oracles.hpp:147-236 ProblemFactory restated
with numpy's RNG: cameras on a 2-4 radius ring looking at a point cluster,
a unit-focal 'normalized' variant, every node referenced by an edge)."""
import numpy as np

from paper_2112_01349_b200 import BAProblem


def _angle_axis(R):
    # rotation matrix -> angle-axis (principal log), generic branch suffices here
    c = np.clip((np.trace(R) - 1) / 2, -1, 1)
    th = np.arccos(c)
    if th < 1e-12:
        return np.zeros(3)
    w = np.array([R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1]]) / (2 * np.sin(th))
    return th * w


class ProblemFactory:
    def __init__(self, seed):
        self.rng = np.random.default_rng(seed)

    def u(self, lo, hi, size=None):
        return self.rng.uniform(lo, hi, size)

    def random_camera(self, normalized=False):
        ang, rad = self.u(0, 2 * np.pi), self.u(2.0, 4.0)
        center = np.array([rad * np.cos(ang), rad * np.sin(ang), self.u(-0.5, 0.5)])
        cz = center / np.linalg.norm(center)
        right = np.cross([0, 0, 1.0], cz)
        right /= np.linalg.norm(right)
        R = np.stack([right, np.cross(cz, right), cz])
        aa = _angle_axis(R) + self.u(-0.05, 0.05, 3)
        t = -(R @ center) + self.u(-0.05, 0.05, 3)
        if normalized:
            f, k1, k2 = self.u(1.0, 3.0), self.u(-0.3, 0.3), self.u(-0.2, 0.2)
        else:
            f, k1, k2 = self.u(500.0, 1500.0), self.u(-0.1, 0.1), self.u(-0.05, 0.05)
        return np.concatenate([aa, t, [f, k1, k2]])

    def random_point(self, normalized=False):
        return self.u(-1.2, 1.2, 3) * np.array([1, 1, 0.8 / 1.2]) if normalized else self.u(-0.3, 0.3, 3)

    def random_problem(self, cameras, points, edges, normalized=False, dtype=np.float64):
        cams = np.stack([self.random_camera(normalized) for _ in range(cameras)])
        pts = np.stack([self.random_point(normalized) for _ in range(points)])
        cid = np.array([e if e < cameras else self.rng.integers(0, cameras) for e in range(edges)], np.int32)
        pid = np.array([e if e < points else self.rng.integers(0, points) for e in range(edges)], np.int32)
        pix = self.u(-1, 1, (edges, 2)) if normalized else self.u(-50, 50, (edges, 2))
        return BAProblem.from_arrays(cams, pts, cid, pid, pix, dtype=dtype)
