"""Counter-based draws (API of pyrocell/rng.py:28-88).

uniform_grid evaluates the keyed SplitMix64 stream on the device
(libfirecell fc_uniform_grid) and returns host fp64, bit-identical to the
reference; derive_epoch_seed is the library's host function.
"""
from __future__ import annotations

from enum import IntEnum

import numpy as np

from . import _lib as L


class Channel(IntEnum):
    """rng.py:28-32."""

    IGNITE = 0
    CONTINUE = 1


def uniform_grid(seed: int, t: int, channel, row0: int, col0: int, height: int,
                 width: int) -> np.ndarray:
    """rng.py:55-75 -- draws for the window at (row0, col0)."""
    from .device import uniform_grid_device
    return uniform_grid_device(seed, t, int(channel), row0, col0, height, width).cpu().numpy()


def uniform_draw(seed: int, t: int, row: int, col: int, channel) -> float:
    """rng.py:78-80."""
    return float(uniform_grid(seed, t, channel, row, col, 1, 1)[0, 0])


def derive_epoch_seed(base_seed: int, epoch: int) -> int:
    """rng.py:83-88 (host function of libfirecell)."""
    return int(L.lib().fc_epoch_seed(int(base_seed) & (2**64 - 1), int(epoch) & (2**64 - 1)))
