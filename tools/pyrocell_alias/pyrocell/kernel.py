"""pyrocell.kernel -> paper_2502_18738_b200.kernel (test-harness alias)."""
import sys as _sys

from paper_2502_18738_b200 import kernel as _impl

_sys.modules[__name__] = _impl
