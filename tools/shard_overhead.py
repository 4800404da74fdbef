"""Overlapped row-shard schedule emulated on one GPU (sharded.run_sharded_local:
one stream per shard, device-copy halo on a communication stream) on the
config-3 domain: device time and host enqueue time per window launch,
against the unsharded run.  python tools/shard_overhead.py [world ...]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_18738_b200 as F  # noqa: E402
from paper_2502_18738_b200 import synthetic as S  # noqa: E402
from paper_2502_18738_b200.sharded import RowPartition, RowShard, run_sharded_local  # noqa: E402


def main():
    worlds = [int(a) for a in sys.argv[1:]] or [2, 4]
    n, steps = 16384, 1000
    e = S.make_environment_torch(n, n, seed=3)
    init = torch.as_tensor(S.random_blocks(n, n, 8, 5, seed=3).astype(np.uint8), device="cuda")
    dl = F.DeviceLandscape.from_elevation(e["elevation"], e["wind_speed"], e["wind_direction"],
                                          e["canopy"], e["density"])
    b = F.FireBatch((n, n), 1, max_steps=steps)
    b.set_params(F.pack_params(0.045, 0.131, 0.078, 0.58, 0.3))
    b.set_seeds([3])
    for k in (1, 4, 8):
        b.reset(init)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        b.run(dl, steps, window=k)
        e1.record()
        host = time.perf_counter() - t0
        torch.cuda.synchronize()
        print(f"unsharded k={k}: device {e0.elapsed_time(e1):.2f} ms, host enqueue {1e3 * host:.2f} ms")
    ref = b.unpack()
    for world in worlds:
        shards = []
        for r in range(world):
            sh = RowShard(RowPartition(n, world, r), e["elevation"], e["wind_speed"],
                          e["wind_direction"], e["canopy"], e["density"], init, max_steps=steps)
            sh.batch.set_params(F.pack_params(0.045, 0.131, 0.078, 0.58, 0.3))
            sh.batch.set_seeds([3])
            shards.append(sh)
        for k in (1, 4, 8):
            def one():
                for sh in shards:
                    sh.batch.reset(sh.batch._init_mask)
                run_sharded_local(shards, steps, k)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            one()
            e1.record()
            host = time.perf_counter() - t0
            torch.cuda.synchronize()
            nwin = (steps + k - 1) // k
            print(f"{world} emulated shards k={k}: device {e0.elapsed_time(e1):.2f} ms, host "
                  f"{1e3 * host:.2f} ms ({1e6 * host / nwin / world:.1f} us per shard-window)")
            g = F.CapturedSequence(one)
            torch.cuda.synchronize()
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            print(f"{world} emulated shards k={k}, one CUDA graph: device {e0.elapsed_time(e1):.2f} ms")
            del g
        ok = all(torch.equal(sh.owned(sh.batch.unpack()[0][0]),
                             ref[0][0, sh.part.owned_rows[0]:sh.part.owned_rows[1]]) for sh in shards)
        print(f"{world} shards bytes equal unsharded (k=8 run): {ok}")
        del shards
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
