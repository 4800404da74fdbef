"""CPU test of the peer-halo protocol's host logic (sharded.run_peer,
include/firecell.h fc_peer_halo): with every shard's work executed in the
order it is enqueued, each stream wait finds its neighbours' event numbers
already stored -- the waits never ask for an event that comes later in
another shard's queue, so the protocol cannot deadlock -- and every call
ends with zero flags."""
import pytest

from paper_2502_18738_b200.sharded import RowPartition, run_peer


class _Batch:
    device = None

    def __init__(self, log, name):
        self.log, self.name, self._init_mask = log, name, None

    def reset(self, init):
        self.log.append((self.name, "reset"))


class _Flags:
    def __init__(self):
        self.v = [0, 0]

    def zero_(self):
        self.v = [0, 0]


class _FakeShard:
    """Duck-typed RowShard: signals store into the neighbours' flag lists,
    waits assert the value is already there (sequential execution)."""

    def __init__(self, part, log):
        self.part, self.log = part, log
        self.batch = _Batch(log, part.rank)
        self.peer_flags = _Flags()
        self._peer = type("P", (), {"seq": 0})()
        self.up = self.down = None

    def _peer_signal(self, value):
        self._store(value)

    def _store(self, value):
        if self.up is not None:
            self.up.peer_flags.v[1] = value    # the upper neighbour's word from below
        if self.down is not None:
            self.down.peer_flags.v[0] = value

    def _wait_peers(self, value):
        for present, i in ((self.part.ghost_top, 0), (self.part.ghost_bottom, 1)):
            if present:
                assert self.peer_flags.v[i] >= value, (self.part.rank, i, self.peer_flags.v, value)
        self.log.append((self.part.rank, "wait", value))

    def run_pass(self, n, window, which, attach=None):
        self.log.append((self.part.rank, f"pass{which}", n))
        if which == 2:
            self._store(self._peer.seq)


@pytest.mark.parametrize("world,steps,window,reset", [(2, 70, 8, False), (3, 17, 4, True),
                                                      (5, 9, 1, False), (1, 10, 4, True)])
def test_peer_protocol_orders_events(world, steps, window, reset):
    log = []
    shards = [_FakeShard(RowPartition(32 * 3 * world, world, r), log) for r in range(world)]
    for a, b in zip(shards[:-1], shards[1:]):
        a.down, b.up = b, a
    for call in range(2):
        run_peer(shards, steps, window, reset=reset)
        for sh in shards:
            assert sh.peer_flags.v == [0, 0]
    launches = -(-steps // window)
    for sh in shards:
        mine = [e for e in log if e[0] == sh.part.rank]
        waits = [e[2] for e in mine if e[1] == "wait"]
        # per call: one wait per launch (>= 1, 2, ..) and the closing drain
        if sh.part.ghost_top or sh.part.ghost_bottom:
            assert waits == 2 * (list(range(1, launches + 1)) + [launches + 1])
        assert sum(e[1] == "pass2" for e in mine) == 2 * launches
        assert sum(e[1] == "reset" for e in mine) == (2 if reset else 0)
