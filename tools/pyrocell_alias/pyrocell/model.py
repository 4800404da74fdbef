"""pyrocell.model -> paper_2502_18738_b200.model (test-harness alias)."""
import sys as _sys

from paper_2502_18738_b200 import model as _impl

_sys.modules[__name__] = _impl
