"""A config's engine (its rank-0 shard), a few eager retrieve() calls: with LC_PROF=1 the kernels
print their per-phase timestamps (diagnostics; not a bench number)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_08453_b200 import api  # noqa: E402


def main():
    args = bench.apply_config(bench.parse())
    args.batch = args.batch or 1
    from paper_2603_08453_b200 import shard
    slots = shard.slots_of_rank(0, max(1, args.shards), args.layers, args.kv_heads, args.batch,
                                order="layer")
    eng, qs, setup, codes = bench.build_engine(api, torch, args, slots, 0)
    q = torch.from_numpy(np.ascontiguousarray(qs)).cuda()
    out = torch.zeros_like(q)
    b = api.Budgets(token_budget=args.budget, unit_topk=8, sink_size=16)
    for _ in range(args.steps):
        eng.retrieve(q, b, out=out)
    torch.cuda.synchronize()
    print("device error", eng.device_error())


if __name__ == "__main__":
    main()
