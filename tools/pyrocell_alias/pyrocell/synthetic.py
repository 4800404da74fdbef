"""pyrocell.synthetic -> paper_2502_18738_b200.synthetic with the reference's
center_ignition(size, block) signature (pyrocell/synthetic.py:129-136)."""
from paper_2502_18738_b200 import synthetic as _impl
from paper_2502_18738_b200.synthetic import (flat_landscape, hill_landscape,  # noqa: F401
                                             make_landscape, random_landscape, valley_landscape,
                                             windy_landscape)


def center_ignition(size: int, block: int = 3):
    return _impl.center_ignition(size, size, block)
