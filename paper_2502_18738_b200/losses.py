"""Calibration loss and metrics (API of pyrocell/losses.py:14-86, 89-111).

combined_loss runs the fused device kernel (fc_loss_dense): union-bbox
BCE-with-logits mean + MSE of 4x4 average pools, with the exact dL/dacc.
Jaccard / Manhattan are integer host metrics over host arrays.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence, Tuple

import numpy as np
import torch

POOL_SIZE = 4


@dataclass(frozen=True)
class LossBreakdown:
    """losses.py:17-29."""

    bce_term: float
    mse_term: float
    crop_window: Tuple[int, int, int, int]

    @property
    def total(self) -> float:
        return self.bce_term + self.mse_term


def combined_loss(accumulator, target) -> Tuple[LossBreakdown, np.ndarray]:
    """losses.py:44-86 -> (LossBreakdown, dL/dacc as host fp64)."""
    from .device import loss_dense
    acc = np.asarray(accumulator, dtype=np.float64)
    y = np.asarray(target)
    if y.shape != acc.shape:
        raise ValueError(f"target shape {y.shape} != accumulator {acc.shape}")
    loss, crop, grad = loss_dense(torch.from_numpy(np.ascontiguousarray(acc)),
                                  torch.from_numpy(np.ascontiguousarray(y.astype(bool).astype(np.uint8))))
    l = loss.cpu().numpy()
    c = tuple(int(v) for v in crop.cpu().numpy())
    return LossBreakdown(float(l[2]), float(l[3]), c), grad.cpu().numpy()


def jaccard_index(a, b) -> float:
    """losses.py:89-98 (Eq. 11)."""
    a = np.asarray(a, dtype=bool)
    b = np.asarray(b, dtype=bool)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    union = int(np.count_nonzero(a | b))
    return 1.0 if union == 0 else int(np.count_nonzero(a & b)) / union


def manhattan_distance(counts_a: Sequence[int], counts_b: Sequence[int]) -> int:
    """losses.py:101-106 (Eq. 12)."""
    if len(counts_a) != len(counts_b):
        raise ValueError(f"length mismatch: {len(counts_a)} vs {len(counts_b)}")
    return int(sum(abs(int(x) - int(y)) for x, y in zip(counts_a, counts_b)))
