"""pyrocell.data_io -> paper_2502_18738_b200.data_io (test-harness alias)."""
import sys as _sys

from paper_2502_18738_b200 import data_io as _impl

_sys.modules[__name__] = _impl
