"""Import alias ``pyrocell`` -> paper_2502_18738_b200 (test harness only).

Lets the reference's own test suite (pyrocell 0.1.0, pkg/tests) run
unmodified against the B200 package: every name the reference re-exports
(pyrocell/__init__.py) resolves to this repository's implementation.  The
two subsystems SURVEY.md marks out of scope -- the scikit-learn estimator
and the normalisation-constant fit -- are stand-ins that raise, so only the
tests that exercise them fail (tools/run_reference_suite.py records why).
"""
from paper_2502_18738_b200 import *  # noqa: F401,F403
from paper_2502_18738_b200 import __all__ as _ours, __version__  # noqa: F401

from .estimator import FireSpreadEstimator  # noqa: F401
from .losses import NormCandidate, fit_normalization_constant  # noqa: F401

__all__ = list(_ours) + ["FireSpreadEstimator", "NormCandidate", "fit_normalization_constant"]
