"""Gaussian record layout (pkg/src/vmsplat/gaussians.py:1-33).

A scene is a dense (n, 59) float32 matrix: position 0..2, rotation quaternion
(w, x, y, z) 3..6, linear scales 7..9, opacity 10, 48 SH coefficients 11..58
stored coefficient-major (sh[c * 3 + ch]).  A page is one contiguous byte
range of rows, which is what the device page pool stores verbatim.
"""

from __future__ import annotations

import numpy as np

RECORD_SIZE = 59
RECORD_BYTES = RECORD_SIZE * 4
SH_COEFFS = 16
POS = slice(0, 3)
ROT = slice(3, 7)
SCALE = slice(7, 10)
OPACITY = 10
SH = slice(11, 59)


def padding_records(count: int) -> np.ndarray:
    return np.zeros((count, RECORD_SIZE), dtype=np.float32)


def is_padding(records: np.ndarray) -> np.ndarray:
    return ~np.asarray(records).any(axis=1)


def quat_to_matrix(q) -> np.ndarray:
    """(w, x, y, z) unit quaternion(s) -> rotation matrix, f64, the same
    elementwise arithmetic as gaussians.py:76-96 (host side: used for the
    camera pose that the kernels receive as an argument)."""
    q = np.asarray(q, dtype=np.float64)
    single = q.ndim == 1
    q = q.reshape(-1, 4)
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    m = np.empty((len(q), 3, 3), dtype=np.float64)
    m[:, 0, 0] = 1 - 2 * (y * y + z * z)
    m[:, 0, 1] = 2 * (x * y - w * z)
    m[:, 0, 2] = 2 * (x * z + w * y)
    m[:, 1, 0] = 2 * (x * y + w * z)
    m[:, 1, 1] = 1 - 2 * (x * x + z * z)
    m[:, 1, 2] = 2 * (y * z - w * x)
    m[:, 2, 0] = 2 * (x * z - w * y)
    m[:, 2, 1] = 2 * (y * z + w * x)
    m[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return m[0] if single else m
