"""pyrocell.rng -> paper_2502_18738_b200.rng (test-harness alias)."""
import sys as _sys

from paper_2502_18738_b200 import rng as _impl

_sys.modules[__name__] = _impl
