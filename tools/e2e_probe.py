"""Where the end-to-end (host-buffer) step's time goes: wall time of
lc_retrieve_host, of the same call's pieces, and the Python wrapper cost.
Run on the GPU box: python tools/e2e_probe.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_08453_b200 import api, shard  # noqa: E402
from paper_2603_08453_b200 import _lib as L  # noqa: E402

sys.argv = sys.argv[:1]
args = bench.apply_config(bench.parse())
args.steps = args.steps or 50
bench.resolve_batch(args)
slots = shard.slots_of_rank(0, 1, args.layers, args.kv_heads, args.batch)
eng, qs, _, _ = bench.build_engine(api, torch, args, slots, 0)
b = api.Budgets(token_budget=args.budget, unit_topk=8, sink_size=16)
qh = torch.from_numpy(np.ascontiguousarray(qs)).pin_memory()
oh = torch.zeros_like(qh).pin_memory()
qd = qh.cuda()
od = torch.zeros_like(qd)
N = 50


def wall(fn, n=N):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e6


qn, on = qh.numpy(), oh.numpy()
print("retrieve_host (python wrapper)   %.1f us" % wall(lambda: eng.retrieve_host(qn, b, on)))
bc = b.c()
st = torch.cuda.current_stream().cuda_stream
fn = L.lib().lc_retrieve_host
print("lc_retrieve_host (raw ctypes)    %.1f us" % wall(lambda: fn(eng.h, qn.ctypes.data, bc, 0, on.ctypes.data, st)))
print("device retrieve + sync           %.1f us" % wall(lambda: (eng.retrieve(qd, b, out=od), torch.cuda.synchronize())))
g = torch.cuda.CUDAGraph()
eng.retrieve(qd, b, out=od)
torch.cuda.synchronize()
with torch.cuda.graph(g):
    eng.retrieve(qd, b, out=od)
print("device graph replay + sync       %.1f us" % wall(lambda: (g.replay(), torch.cuda.synchronize())))
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); ev0.record()
for _ in range(N):
    g.replay()
ev1.record(); torch.cuda.synchronize()
print("device graph (events, back to back) %.1f us" % (ev0.elapsed_time(ev1) / N * 1e3))
print("H2D + D2H pinned + sync          %.1f us" % wall(lambda: (qd.copy_(qh, non_blocking=True), oh.copy_(od, non_blocking=True), torch.cuda.synchronize())))
print("empty ctypes call                %.1f us" % wall(lambda: L.lib().lc_last_error()))
