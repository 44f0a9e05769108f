"""Fixtures of proj/tests/test_raster.cpp:12-39 and the reference Rng (math_util.hpp:27-63)."""
import math

import numpy as np

from paper_2604_10982_b200 import Camera, SceneMap

M64 = (1 << 64) - 1


class Rng:
    """splitmix64 + Box-Muller, bit-identical to psimap::Rng (math_util.hpp:27-63)."""

    def __init__(self, seed=0):
        self.state = seed & M64

    def next(self):
        self.state = (self.state + 0x9E3779B97F4A7C15) & M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def uniform(self, lo=None, hi=None):
        u = float(self.next() >> 11) * 2.0 ** -53
        if lo is None:
            return u
        return lo + (hi - lo) * u

    def normal(self):
        u1 = self.uniform()
        u2 = self.uniform()
        if u1 < 1e-300:
            u1 = 1e-300
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)

    def uniform_int(self, n):
        return 0 if n == 0 else self.next() % n

    def unit_quaternion(self):
        q = np.array([self.normal() for _ in range(4)])
        n = math.sqrt((q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3]))
        if n < 1e-12:
            return np.array([1.0, 0, 0, 0])
        return q / n


def front_camera(w=64, h=64, f=100.0):
    """test_raster.cpp:14-18: identity pose looking down +z, principal point on a pixel centre."""
    return Camera.make(np.eye(3), np.zeros(3), f, f, w // 2 - 0.5, h // 2 - 0.5, w, h, 0.1, 100.0)


def facing_surfel(center, s1, s2, opacity, color, quat=(1.0, 0.0, 0.0, 0.0)):
    """test_raster.cpp:20-30 as a 13-double row."""
    return np.array([*center, *quat, s1, s2, opacity, *color], dtype=np.float64)


def scene_of(rows, f_sem=None):
    rows = np.asarray(rows, dtype=np.float64).reshape(-1, 13)
    if f_sem is None:
        f_sem = np.zeros((rows.shape[0], 2))  # facing_surfel gives f_sem = Zero(2)
    return SceneMap(rows, f_sem)
