"""pyrocell.cli -> paper_2502_18738_b200.cli (test-harness alias)."""
import sys as _sys

from paper_2502_18738_b200 import cli as _impl

_sys.modules[__name__] = _impl
