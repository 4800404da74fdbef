"""Peer-memory halo under CUDA-graph replay: three emulated row shards on
one GPU (each on its own stream), the run with reset captured once and
replayed three times; each replay must equal the unsharded run and leave
every flag word at zero.  python tools/peer_graph_check.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_18738_b200 as F
from paper_2502_18738_b200 import synthetic as S
from paper_2502_18738_b200.sharded import RowPartition, RowShard, connect_local_peers, run_peer_local
h, w, steps, world, window = 300, 140, 70, 3, 4
env = S.make_environment(h, w, seed=35)
init = S.random_blocks(h, w, 6, 5, seed=6) | S.center_ignition(h, w)
params = F.pack_params(0.06, 0.12, 0.08, 0.6, 0.45)
ref = F.FireBatch((h, w), 1, max_steps=steps); ref.set_params(params); ref.set_seeds([79]); ref.reset(init)
ref.run(F.DeviceLandscape.from_environment(env), steps, window=window)
rb, rd = ref.unpack()
shards = []
for r in range(world):
    sh = RowShard(RowPartition(h, world, r), env.elevation, env.wind_speed, env.wind_direction,
                  env.canopy, env.density, init, max_steps=steps)
    sh.batch.set_params(params); sh.batch.set_seeds([79]); shards.append(sh)
connect_local_peers(shards)
g = F.CapturedSequence(lambda: run_peer_local(shards, steps, window=window, reset=True))
for rep in range(3):
    g.replay(); torch.cuda.synchronize()
    gb = torch.cat([sh.owned(sh.batch.unpack()[0][0]) for sh in shards])
    print("replay", rep, torch.equal(gb, rb[0]), [int(sh.peer_flags.abs().sum()) for sh in shards])
