"""Cosine triangle bounds (host mirror; the device versions live in csrc/spkm.cu).

For unit x, z, y with a = <x,z>, b = <z,y> (reference geometry.py:1-77,
paper Eqs. 4-10):
    a*b - sqrt((1-a^2)(1-b^2)) <= <x,y> <= a*b + sqrt((1-a^2)(1-b^2))
The device kernels evaluate these in float64 and then round the stored
float32 bound outward (down for lower bounds, up for upper bounds).
"""

import numpy as np


def clamp_cos(t):
    return np.clip(t, -1.0, 1.0)


def _sin(t):
    return np.sqrt(np.maximum(0.0, 1.0 - t * t))


def cos_lower_bound(a, b):
    return clamp_cos(a * b - _sin(a) * _sin(b))


def cos_upper_bound(a, b):
    return clamp_cos(a * b + _sin(a) * _sin(b))


def update_lower_bound(l, p):
    return cos_lower_bound(l, p)


def update_upper_bound(u, p):
    return cos_upper_bound(u, p)


def hamerly_upper_update(u, p_min):
    """u + sin(u) sin(p_min): dominates every per-cluster update with p >= p_min."""
    return clamp_cos(u + _sin(u) * _sin(p_min))


def half_angle_cc(s):
    return np.sqrt(np.maximum(0.0, (s + 1.0) / 2.0))


def arccos_triangle_oracle(a, b):
    """cos(arccos a + arccos b) -- trigonometric cross-check, tests only."""
    return np.cos(np.arccos(clamp_cos(a)) + np.arccos(clamp_cos(b)))
