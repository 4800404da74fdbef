"""pyrocell.tape -> paper_2502_18738_b200.tape (test-harness alias)."""
import sys as _sys

from paper_2502_18738_b200 import tape as _impl

_sys.modules[__name__] = _impl
