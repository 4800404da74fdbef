"""pyrocell.calibration -> paper_2502_18738_b200.calibration (test-harness alias)."""
import sys as _sys

from paper_2502_18738_b200 import calibration as _impl

_sys.modules[__name__] = _impl
