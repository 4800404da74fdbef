"""pyrocell.losses -> paper_2502_18738_b200.losses, plus stand-ins for the
normalisation-constant fit (losses.py:109-160), out of scope."""
from enum import Enum

from paper_2502_18738_b200.losses import *  # noqa: F401,F403
from paper_2502_18738_b200.losses import LossBreakdown, combined_loss  # noqa: F401

_WHY = "normalisation-constant fit: out of scope for the B200 hot path (SURVEY.md 2)"


class NormCandidate(Enum):
    EXP_BASE = "exp_base"
    POWER = "power"
    TANH = "tanh"


def fit_normalization_constant(candidate):
    raise NotImplementedError(_WHY)


def fit_all_candidates():
    raise NotImplementedError(_WHY)


def _candidate_values(candidate, c, x):
    raise NotImplementedError(_WHY)
