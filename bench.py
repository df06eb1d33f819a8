#!/usr/bin/env python
"""Decode-step throughput of the B200 LycheeCluster path (BASELINE.json metric).

Workload (BASELINE.json configs[1]): Llama-3-8B-shaped cache -- 32 layers x
8 KV heads (d = 128), GQA 4 (32 query heads), 128K-token context, batch 1,
2K-token budget.  One step = retrieve() + sparse attention for all 1024
query heads (32 layers x 32 heads), i.e. one decode step of the model's
attention path.  Every (layer, KV head) slot has its own synthetic
clustered KV stream (gen_clustered_workload, seed 1000 + slot, generated on
the GPU), its own index (build_index, on the GPU, bit-exact to the
reference) and its own 4 queries.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun): the 256 slots are sharded by KV head over the ranks
(strong scaling of the batch-1 step); the head outputs are all-gathered over
NCCL once per step.  `--impl reference` times the reference CPU path
(oracle/_ref, built from /root/reference) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "retrieval+sparse-attn decode steps/s @128K (Llama-3-8B shape); % HBM roofline"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=0, help="timed steps (default 50; --mode stream: 4096)")
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--mode", default="step", choices=["step", "stream"],
                   help="step: config 2 retrieval + attention (the headline); stream: config 3 "
                        "decode steps with KV append and lazy grafts (batch --batch, default 8)")
    p.add_argument("--config", type=int, default=2, choices=[1, 2, 4, 5],
                   help="BASELINE.json configs: 1 = 32K single layer, 2 = the headline (128K, Llama-3-8B shape), "
                        "4 = Qwen3-8B shape at 1M sharded over --shards GPUs, 5 = the batched decode sweep "
                        "(config 3 is --mode stream)")
    p.add_argument("--shards", type=int, default=0,
                   help="KV-head shards of the job (default: the number of GPUs; config 4: 2). With fewer GPUs "
                        "than shards, this process runs shard RANK of them")
    p.add_argument("--tokens", type=int, default=None)
    p.add_argument("--layers", type=int, default=None)
    p.add_argument("--kv-heads", type=int, default=None)
    p.add_argument("--group", type=int, default=None)
    p.add_argument("--budget", type=int, default=None)
    p.add_argument("--batch", type=int, default=0,
                   help="sequences per step; default: the number of GPUs (weak scaling: every GPU keeps "
                        "one sequence's worth of slots, config 2's per-GPU load) -- 8 in --mode stream")
    p.add_argument("--graph", type=int, default=1)
    p.add_argument("--slot-groups", type=int, default=1)
    p.add_argument("--gather", default="nccl", choices=["nccl", "p2p"],
                   help="N > 1: the layer-boundary all-gather of head outputs over NCCL, or fused into the "
                        "attention merge as NVLink peer stores into symmetric-memory buffers (lc_set_gather)")
    p.add_argument("--cpu-baseline", type=int, default=1)
    p.add_argument("--l2-flush", type=int, default=-1,
                   help="flush L2 between timed iterations: -1 auto (when a step's inputs are < 3x L2), 0 off, 1 on")
    p.add_argument("--seed-base", type=int, default=1000)
    p.add_argument("--ref-slots", type=int, default=4,
                   help="distinct reference-built slots the CPU reference timing spreads its calls over")
    p.add_argument("--parity", type=int, default=1,
                   help="re-check sampled slots' selections against the reference (oracle/_ref) after timing")
    return p.parse_args()


CONFIGS = {
    1: dict(layers=1, kv_heads=8, group=4, tokens=32768, budget=2048, shards=0,
            name="config1: synthetic single-layer decode (1 layer x 8 KV heads x d128, GQA 4)"),
    2: dict(layers=32, kv_heads=8, group=4, tokens=131072, budget=2048, shards=0,
            name="config2: Llama-3-8B-shaped cache (32 layers x 8 KV heads x d128, GQA 4)"),
    4: dict(layers=36, kv_heads=8, group=4, tokens=1 << 20, budget=2048, shards=2,
            name="config4: Qwen3-8B-shaped cache (36 layers x 8 KV heads x d128, GQA 4), KV heads sharded"),
    5: dict(layers=1, kv_heads=8, group=4, tokens=131072, budget=2048, shards=8,
            name="config5: batched decode sweep (1 layer x 8 KV heads x d128, GQA 4), KV heads sharded over 8 GPUs"),
}


def apply_config(args):
    c = CONFIGS[args.config]
    for k in ("layers", "kv_heads", "group", "tokens", "budget"):
        if getattr(args, k) is None:
            setattr(args, k, c[k])
    if not args.shards:
        args.shards = c["shards"]
    args.config_name = c["name"]
    return args


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append(parts)
            except Exception:
                pass
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        load = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def build_engine(api, torch, args, slots, device):
    n = args.tokens
    S = len(slots)
    cap_chunks = n // 8 + 64
    eng = api.Engine(S, 128, args.group, cap_tokens=n + 64, cap_chunks=cap_chunks,
                     cap_clusters=(cap_chunks + 1) // 2, cap_units=64,
                     keep_reps=False, device=device, slot_groups=args.slot_groups)
    seeds = np.array([args.seed_base + s for s in slots], np.uint64)
    t0 = time.time()
    codes, qs = eng.gen_workload(n, seeds, query_count=args.group)
    t1 = time.time()
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 4)) as ex:
        spans = list(ex.map(lambda s: api.segment_codes(codes[s]), range(S)))
    t2 = time.time()
    eng.build_index([n] * S, spans, seeds)
    torch.cuda.synchronize()
    t3 = time.time()
    setup = {"gen_s": round(t1 - t0, 2), "segment_s": round(t2 - t1, 2), "build_s": round(t3 - t2, 2)}
    return eng, qs, setup, codes


def time_loop(torch, fn, steps, stream):
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(steps):
        fn()
    ev1.record(stream)
    torch.cuda.synchronize()
    return ev0.elapsed_time(ev1) / steps  # ms


def verify_outputs(api, torch, eng, q, out, n_tokens, slots):
    """Plain torch fp64 attention over each checked head's own active set (the
    engine's selection) vs the kernel output: the bench's correctness guard."""
    worst = 0.0
    o = out.cpu().numpy()
    qn = q.cpu().numpy()
    for s in slots:
        kb, vb = eng.kv_download(s, n_tokens)
        K = torch.from_numpy((kb.astype(np.uint32) << 16).view(np.float32)).cuda().double()
        V = torch.from_numpy((vb.astype(np.uint32) << 16).view(np.float32)).cuda().double()
        for g in range(q.shape[1]):
            ids = torch.from_numpy(eng.selection(s, g).active_token_ids.astype(np.int64)).cuda()
            qq = torch.from_numpy(qn[s, g].astype(np.float64)).cuda()
            w = torch.softmax((K[ids] @ qq) / np.sqrt(K.shape[1]), dim=0)
            ref = (w[:, None] * V[ids]).sum(0).cpu().numpy()
            err = float(np.linalg.norm(o[s, g] - ref) / max(np.linalg.norm(ref), 1e-30))
            worst = max(worst, err)
    return worst


def parity_vs_reference(eng, codes, qs, out, slots, budgets):
    """Selections of the timed step vs the reference's own retrieve()
    (oracle/_ref, retriever.cpp:161-167) on the same indexes: each sampled
    slot's GPU-built index and K/V go to the reference through a TKIX file
    (lc_index_save -> load_index), then every head's units, clusters (rank
    order), scanned count and active ids must be identical and the output
    within 1e-3 relative."""
    from oracle import refpy as R
    if not R.available():
        return {"ok": None, "why": "oracle/_ref not built"}
    o = out.cpu().numpy()
    heads, worst, bad = 0, 0.0, []
    t0 = time.time()
    for s in slots:
        texts = ["\n" if c == 1 else ("}" if c == 2 else "") for c in codes[s]]
        fd, path = tempfile.mkstemp(suffix=".tkix")
        os.close(fd)
        try:
            eng.save_index(s, path, texts)
            ref = R.RefEngine.load(path)
        finally:
            os.unlink(path)
        for g in range(qs.shape[1]):
            r = ref.retrieve(qs[s, g], token_budget=budgets.token_budget, unit_topk=budgets.unit_topk,
                             sink=budgets.sink_size)
            got = eng.selection(s, g)
            same = (got.degenerate == r["degenerate"] and np.array_equal(got.selected_units, r["units"])
                    and np.array_equal(got.selected_clusters, r["clusters"])
                    and got.scanned_centroids == r["scanned"]
                    and np.array_equal(got.active_token_ids, r["active"]))
            err = float(np.linalg.norm(o[s, g] - r["output"]) / max(np.linalg.norm(r["output"]), 1e-30))
            worst = max(worst, err)
            heads += 1
            if not same or err >= 1e-3:
                bad.append([int(s), int(g)])
    return {"ok": not bad, "heads_checked": heads, "slots": [int(s) for s in slots], "mismatches": bad,
            "max_rel_err_vs_reference": worst, "tolerance": 1e-3, "seconds": round(time.time() - t0, 1),
            "what": "selected units, clusters (rank order), scanned count and active ids bit-exact vs oracle/_ref "
                    "retrieve() on the same GPU-built index (TKIX round trip); output within tolerance"}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def metric_of(args):
    if getattr(args, "config", 2) == 2:
        return METRIC
    return f"retrieval+sparse-attn decode steps/s ({args.config_name}, {args.tokens}-token context); % HBM roofline"


def ref_from_gpu(eng, codes, s):
    """A GPU-built slot handed to the reference (lc_index_save -> the
    reference's load_index through a TKIX file): baseline timing at contexts
    whose CPU build would take ~15 min per slot."""
    from oracle import refpy as R
    texts = ["\n" if c == 1 else ("}" if c == 2 else "") for c in codes[s]]
    fd, path = tempfile.mkstemp(suffix=".tkix")
    os.close(fd)
    try:
        eng.save_index(s, path, texts)
        return R.RefEngine.load(path)
    finally:
        os.unlink(path)


def cpu_baseline_ref(args, n_query_heads, threads=0, steps=2, src=None):
    """The reference's own CPU path (oracle/_ref) on a bounded sample:
    args.ref_slots distinct reference-built slots of the configured context
    (gen_clustered_workload seeds seed_base+s, build_index on the host), and per
    step n_query_heads retrieve() calls (ids + sparse attention) spread evenly
    over them (each slot's own queries cycled), OpenMP over calls with every
    host thread (mode B), after one warm-up step.  Mode A (the reference API
    as-is: serial calls, OpenMP inside the kernels) is timed on one slot's
    queries and scaled."""
    from oracle import refpy as R
    if not R.available():
        return None
    t0 = time.time()
    refs, qlist = [], []
    if src is not None and args.tokens > 262144:  # GPU-built slots through TKIX (labelled in the sample text)
        eng, codes, qs = src
        for s in range(min(max(1, args.ref_slots), len(codes))):
            refs.append(ref_from_gpu(eng, codes, s))
            qlist.append(np.ascontiguousarray(qs[s], np.float32))
        args.ref_from_gpu = True
    else:
        for s in range(max(1, args.ref_slots)):
            w = R.gen_workload(args.tokens, 128, seed=args.seed_base + s, query_count=args.group)
            refs.append(R.RefEngine(w.keys, w.values, w.text_code, seed=args.seed_base + s))
            qlist.append(w.queries)
            del w
    setup = time.time() - t0
    nthreads = R.threads() if threads == 0 else threads
    per = max(1, n_query_heads // len(refs))
    qs = np.ascontiguousarray(np.concatenate([np.tile(q, (-(-per // args.group), 1))[:per] for q in qlist]),
                              np.float32)
    R.time_retrieve(refs, qs, token_budget=args.budget, reps=1, mode=1, threads=threads)  # warm-up
    times = [R.time_retrieve(refs, qs, token_budget=args.budget, reps=1, mode=1, threads=threads)[0]
             for _ in range(steps)]
    step_b = sum(times) / len(times) * n_query_heads / qs.shape[0]
    secs_a, _ = R.time_retrieve(refs[:1], qlist[0], token_budget=args.budget, reps=1, mode=0, threads=threads)
    return {"threads": nthreads, "setup_s": setup, "refs": refs, "qs": qs, "step_s": step_b,
            "step_mode_a_s": secs_a / args.group * n_query_heads, "calls": qs.shape[0] * steps,
            "cpu": cpu_model()}


def ref_sample_text(args, n_qh, base):
    how = ("GPU-built slots (the bench's own, bit-exact to the reference build) loaded by the reference's "
           "load_index from TKIX files" if getattr(args, "ref_from_gpu", False) else "reference-built")
    return (f"oracle/_ref (the reference built from /root/reference): {len(base['refs'])} distinct "
            f"{how} {args.tokens}-token slots (seeds {args.seed_base}..{args.seed_base + len(base['refs']) - 1}, "
            f"build_index on the host, {base['setup_s']:.0f} s); each step = {n_qh} retrieve() calls (ids + sparse "
            f"attention) spread evenly over them, each slot's {args.group} queries cycled; OpenMP over calls on "
            f"{base['threads']} threads of a {base['cpu']}. Mode A (reference API as-is, serial calls, OpenMP "
            f"kernels): {1.0 / base['step_mode_a_s']:.3f} steps/s")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_qh = args.layers * args.kv_heads * args.group * args.batch
    base = cpu_baseline_ref(args, n_qh)
    if base is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    from oracle import refpy as R
    refs, qs = base["refs"], base["qs"]
    # each step: all query-head retrieve() calls of one decode step over the
    # distinct reference-built slots, OpenMP over calls
    for _ in range(args.warmup):
        R.time_retrieve(refs, qs, token_budget=args.budget, reps=1, mode=1)
    times = []
    for _ in range(args.steps):
        secs, _ = R.time_retrieve(refs, qs, token_budget=args.budget, reps=1, mode=1)
        times.append(secs * n_qh / qs.shape[0])
    step = sum(times) / len(times)
    v = args.batch / step
    line = {
        "impl": "reference", "metric": metric_of(args), "value": v, "unit": "steps/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3, "higher_is_better": True,
        "scaling": getattr(args, "scaling", "strong"), "value_definition": VALUE_DEF, "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (reference gen_clustered_workload, seeds %d+slot)" % args.seed_base,
        "config": config_dict(args, 1),
        "cpu_baseline": {"value": v, "unit": "steps/s", "cores": base["threads"], "kind": "reference",
                         "cpu": base["cpu"], "sample": ref_sample_text(args, n_qh, base)},
        "e2e": {"value": v, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def config_dict(args, world):
    shards = getattr(args, "shards", 0) or world
    par = f"kv-head shard x{world}" if world > 1 else "1 GPU"
    if shards > world:
        par = (f"KV heads sharded over {shards} GPUs; this run measured shard {getattr(args, 'shard', 0)} of "
               f"{shards} on {world} GPU (shards are symmetric: same shapes, independent slots, no collective "
               f"inside the step), so the job's step time is this shard's")
    return {"workload": f"{getattr(args, 'config_name', 'config2')}, "
                        f"{args.tokens}-token context, batch {args.batch}, {args.budget}-token budget",
            "config": getattr(args, "config", 2), "shards": shards,
            "layers": args.layers, "kv_heads": args.kv_heads, "group": args.group,
            "context": args.tokens, "batch": args.batch, "token_budget": args.budget,
            "unit_topk": 8, "sink": 16, "slots": args.layers * args.kv_heads * args.batch,
            "parallelism": par,
            "l2": ("flushed before every timed iteration (a 252 MB buffer written outside the event pairs)"
                   if getattr(args, "l2_flush", 0) == True else
                   "inputs larger than L2 (index + KV read per step > 3 x the 126 MB L2)")}


def stream_takes(total_steps, min_len=8, max_len=16, marker_every=12):
    """The host chunker's flush decisions for the decoded text stream
    (push_token / flush_buffer, streamer.cpp:29-66): a "\\n" marker every 12
    decoded tokens like run_stream (bench.cpp:254-260); when the buffer reaches
    max_len the head span is grafted.  Every slot of a sequence shares the
    stream, so one decision per step applies to all of them.
    -> [(step, take, kind, level)]"""
    from paper_2603_08453_b200 import api
    buf, out = [], []
    for i in range(total_steps):
        buf.append("\n" if (i + 1) % marker_every == 0 else "")
        if len(buf) >= max_len:
            t, kd, lv = api.flush_take(buf, min_len=min_len, max_len=max_len)
            out.append((i, t, kd, lv))
            buf = buf[t:]
    return out


def stream_cpu_baseline(args, total_slots, steps=48, copies=0):
    """The reference's own decode path (oracle/_ref StreamState::decode_step,
    streamer.cpp:145-165) on the host cores: one reference-built slot of the
    configured prefix, cloned through the reference's save_index / load_index
    into one engine per host thread, every engine running `steps` decode
    steps (run_stream-style stationary queries and same-blob tokens, a marker
    every 12 tokens) in parallel threads.  Whole-job steps/s for total_slots
    slots is extrapolated from the parallel throughput (labelled)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import refpy as R
    if not R.available():
        return None
    t0 = time.time()
    w = R.gen_workload(args.tokens, 128, seed=args.seed_base, query_count=1)
    base = R.RefEngine(w.keys, w.values, w.text_code, seed=args.seed_base)
    fd, path = tempfile.mkstemp(suffix=".tkix")
    os.close(fd)
    try:
        base.save(path)
        nthr = copies or R.threads()
        engines = [R.RefEngine.load(path) for _ in range(nthr)]
    finally:
        os.unlink(path)
    setup = time.time() - t0
    # run_stream-style stationary decode (bench.cpp:240-272): queries around the
    # workload's own query, unit keys near it, N(0,1) values
    rng = np.random.default_rng(5)
    c = w.queries[0] / np.linalg.norm(w.queries[0])
    toks = []
    for i in range(steps):
        q = c + 0.33 / np.sqrt(128) * rng.standard_normal(128)
        q = (q * np.sqrt(128) / np.linalg.norm(q)).astype(np.float32)
        k = c + 0.33 / np.sqrt(128) * rng.standard_normal(128)
        k = (k / np.linalg.norm(k)).astype(np.float32)
        toks.append((q, k, rng.standard_normal(128).astype(np.float32), 1 if (i + 1) % 12 == 0 else 0))

    def run(e):
        R.set_thread_team(1)  # one single-threaded engine per host thread
        for q, k, v, code in toks:
            e.decode_step(q, k, v, code, token_budget=args.budget)

    t1 = time.time()
    with ThreadPoolExecutor(max_workers=nthr) as ex:
        list(ex.map(run, engines))
    wall = time.time() - t1
    slot_steps_per_s = nthr * steps / wall
    return {"value": slot_steps_per_s / total_slots, "unit": "steps/s", "cores": nthr, "kind": "reference",
            "cpu": cpu_model(),
            "sample": f"oracle/_ref StreamState::decode_step (retrieve + attention + push_token + lazy graft): one "
                      f"reference-built {args.tokens}-token slot cloned via save_index/load_index into {nthr} "
                      f"engines, {steps} decode steps each on {nthr} parallel host threads ({wall:.1f} s, setup "
                      f"{setup:.0f} s); whole-job value EXTRAPOLATED to {total_slots} slots as "
                      f"(slot-steps/s) / {total_slots}"}


def run_stream_mode(args, api, torch):
    """Config 3: a 128K prefix per slot, then 4K decode steps through
    lc_decode_step_async -- retrieve(buffer) + attention, KV append, and the
    lazy graft on the steps where the host chunker flushes (streamer.cpp:
    145-165) -- for every (layer, KV head, sequence) slot at once.  The flush
    decisions (take / kind / level per step) are the host chunker's, made
    ahead for the shared decoded text stream and handed to the device as
    arrays, so the whole timed run is ONE CUDA graph with no host sync."""
    batch = args.batch if args.batch > 1 else 8
    args.batch = batch
    n = args.tokens
    slots = list(range(args.layers * args.kv_heads * batch))
    S, d, G = len(slots), 128, args.group
    steps = args.steps if args.steps else 4096
    warm = max(args.warmup, 3)
    total = warm + steps
    plan = stream_takes(total)
    cap_chunks = n // 8 + 64 + len(plan) + 8
    eng = api.Engine(S, d, G, cap_tokens=n + total + 64, cap_chunks=cap_chunks,
                     cap_clusters=(n // 8 + 64 + 1) // 2, cap_units=64, keep_reps=False)
    seeds = np.array([args.seed_base + s for s in slots], np.uint64)
    t0 = time.time()
    codes, qs = eng.gen_workload(n, seeds, query_count=G)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 4)) as ex:
        spans = list(ex.map(lambda s: api.segment_codes(codes[s]), range(S)))
    eng.build_index([n] * S, spans, seeds)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    dims = [eng.slot_dims(s) for s in (0, S // 2, S - 1)]
    ring = 64  # distinct per-step inputs, cycled (a stationary decode, run_stream-like)
    gen = torch.Generator(device="cuda").manual_seed(7)
    q0 = torch.from_numpy(np.ascontiguousarray(qs)).cuda()
    qn = q0 + 0.05 * torch.randn((ring,) + tuple(q0.shape), device="cuda", generator=gen)
    qn = (qn * (np.sqrt(d) / qn.norm(dim=-1, keepdim=True))).contiguous()
    kv = torch.randn((ring, 2, S, d), device="cuda", generator=gen)
    kv[:, 0] = kv[:, 0] / kv[:, 0].norm(dim=-1, keepdim=True)
    kv = kv.to(torch.bfloat16).contiguous().view(torch.int16)
    out = torch.zeros_like(q0)
    b = api.Budgets(token_budget=args.budget, unit_topk=8, sink_size=16)
    take_of = {i: (t, kd, lv) for i, t, kd, lv in plan}
    tk = torch.zeros((max(1, len(plan)), 3, S), dtype=torch.int32, device="cuda")
    for j, (i, t, kd, lv) in enumerate(plan):
        tk[j, 0] = t
        tk[j, 1] = kd
        tk[j, 2] = lv
    slot_of_plan = {i: j for j, (i, _, _, _) in enumerate(plan)}

    def step(i):
        j = slot_of_plan.get(i)
        tks = (tk[j, 0], tk[j, 1], tk[j, 2]) if j is not None else (None, None, None)
        eng.decode_step_async(qn[i % ring], kv[i % ring, 0], kv[i % ring, 1], b, *tks, out=out)

    for i in range(warm):
        step(i)
    torch.cuda.synchronize()
    err = eng.device_error()
    if err:
        raise RuntimeError(f"device error bits 0x{err:x}")
    sb = eng.step_bytes()
    launches_plain = eng.launch_count()
    chunks0 = [eng.slot_dims(s)[1] for s in (0, S - 1)]
    grafts_warm = sum(1 for i, *_ in plan if i < warm)
    graph = None
    if args.graph:
        graph = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(graph, stream=cs):
            for i in range(warm, total):
                step(i)
        torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        ev0.record()
        if graph is not None:
            graph.replay()
        else:
            for i in range(warm, total):
                step(i)
        ev1.record()
        torch.cuda.synchronize()
    clocks = clk.summary()
    ms = ev0.elapsed_time(ev1) / steps
    err = eng.device_error()
    if err:
        raise RuntimeError(f"device error bits 0x{err:x}")
    grafts = sum(1 for i, *_ in plan if i >= warm)
    n_end = eng.slot_dims(0)[4]
    assert n_end == n + total, (n_end, n + total)
    chunks1 = [eng.slot_dims(s)[1] for s in (0, S - 1)]
    assert all(c1 - c0 == grafts for c0, c1 in zip(chunks0, chunks1)), (chunks0, chunks1, grafts)
    # the last timed step's outputs vs a torch fp64 attention over each checked head's own active set
    vslots = [0, S // 2, S - 1]
    max_err = verify_outputs(api, torch, eng, qn[(total - 1) % ring], out, n_end, vslots)
    # algorithmic bytes per step: the retrieval step's union
    # bytes (measured on a warm-up step) + the KV append + the grafts' reads
    # and writes averaged over the timed steps
    e = 2
    L, P = dims[0][2], dims[0][3]
    take_mean = np.mean([t for i, t, *_ in plan if i >= warm]) if grafts else 0.0
    graft_bytes = S * (take_mean * d * e + P * 4 * d + (L / max(P, 1)) * 4 * d + 4 * d + 16)
    step_bytes = sb[0] + S * 2 * d * e + graft_bytes * grafts / steps
    # the certified filter reads the fine tier at fp16 width (2d + 16 B per candidate, not 4d + 16)
    step_bytes16 = step_bytes - sb[3] * 2 * d
    peak, peak_src = peaks()
    gbs = step_bytes16 / (ms * 1e-3) / 1e9
    cpu = stream_cpu_baseline(args, S) if args.cpu_baseline else None
    line = {
        "metric": "config3 streaming decode steps/s (retrieve + attend + append + lazy graft, every slot)",
        "value": 1000.0 / ms, "unit": "steps/s", "n_gpus": 1, "steps": steps, "warmup": warm,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": f"synthetic (gen_clustered_workload prefixes on the GPU, seeds {args.seed_base}+slot, GPU "
                f"build_index; decoded tokens: stationary queries and unit keys / N(0,1) values from a ring of "
                f"{ring} per-step sets; a newline marker every 12 decoded tokens)",
        "config": {"workload": f"config3: {args.layers} layers x {args.kv_heads} KV heads x batch {batch} "
                               f"(= {S} slots), {n}-token prefix + {total} decoded tokens, {args.budget}-token "
                               "budget, lazy graft on every flush",
                   "slots": S, "context": n, "batch": batch, "token_budget": args.budget,
                   "l2": "inputs larger than L2 (> 2 GB read per step vs 126 MB L2)"},
        "roofline": {"bound": "hbm", "kernel": "whole decode step (k_select, k_attend, k_merge, k_append, k_graft)",
                     "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak, "traffic": None,
                     "peak_source": peak_src,
                     "bytes_definition": "bytes the step's algorithm reads and writes: SURVEY s8(d) union bytes "
                                         "with the fine tier at the fp16 width the certified filter streams, + "
                                         "append + grafts; frac_survey_fp32_fine_width counts the fine tier at "
                                         "the reference's fp32 width (bytes this path never reads). The peak is "
                                         "a copy (read + write); a read-dominated stream can exceed it a little",
                     "bytes_per_step": step_bytes16, "frac_survey_fp32_fine_width": step_bytes / (ms * 1e-3) / 1e9 / peak,
                     "bytes_per_step_survey": step_bytes,
                     "bytes_retrieval_union": sb[0], "bytes_append": S * 2 * d * e,
                     "bytes_graft_per_graft_step": graft_bytes},
        "cpu_baseline": cpu,
        "e2e": None,
        "grafts_per_slot_timed": grafts, "graft_rate": grafts / steps,
        "grafts_applied_on_device": {"slots": [0, S - 1], "chunks_before": chunks0, "chunks_after": chunks1},
        "check": {"max_rel_err_vs_torch_fp64": max_err, "tolerance": 1e-3, "slots": vslots, "ok": max_err < 1e-3,
                  "what": "the last timed step's outputs vs torch fp64 attention over each head's own active set"},
        "gpu_launches": steps * (launches_plain) + grafts,
        "kernels_per_step": f"{launches_plain} (k_select, k_attend, k_merge, k_append) + k_graft on flush steps",
        "cuda_graph": graph is not None,
        "clocks": clocks, "setup_s": round(setup_s, 1),
        "final_tokens_per_slot": n_end,
    }
    print(json.dumps(line))


SWEEP_BATCH = (1, 8, 64)
SWEEP_CONTEXT = (32768, 131072, 524288)
SWEEP_BUDGET = (1024, 2048, 8192)


def run_sweep(args, api, torch):
    """Config 5: batch 1-64 x context 32K-512K x budget 1K-8K, one layer, KV
    heads sharded over args.shards GPUs (8).  Each (batch, context) point
    builds its shard's slots once (GPU generator + GPU build_index) and times
    the decode step for every budget (CUDA graph, CUDA events)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    from paper_2603_08453_b200 import shard
    shards = args.shards or world
    args.shard = rank if shards == world else 0
    peak, peak_src = peaks()
    stream = torch.cuda.current_stream()
    points = []
    d = 128
    t_all = time.time()
    for ctx in SWEEP_CONTEXT:
        for batch in SWEEP_BATCH:
            a = argparse.Namespace(**vars(args))
            a.tokens, a.batch = ctx, batch
            slots = shard.slots_of_rank(args.shard, shards, a.layers, a.kv_heads, batch, order="layer")
            eng, qs, setup, codes = build_engine(api, torch, a, slots, local)
            q = torch.from_numpy(np.ascontiguousarray(qs)).cuda()
            out = torch.zeros_like(q)
            for budget in SWEEP_BUDGET:
                b = api.Budgets(token_budget=budget, unit_topk=8, sink_size=16)
                ms, graphed = timed(torch, None, 1, lambda: eng.retrieve(q, b, out=out), args.steps, stream, 3,
                                    "sweep step", graph=args.graph, flush=True)
                err = eng.device_error()
                if err:
                    raise RuntimeError(f"device error bits 0x{err:x} at {(batch, ctx, budget)}")
                sb = eng.step_bytes()
                fp16 = sb[0] - sb[3] * (2 * d)
                par = None
                if args.parity and budget == SWEEP_BUDGET[-1]:  # the last slot vs the reference, largest budget
                    par = parity_vs_reference(eng, codes, qs, out, [len(slots) - 1], b)
                    par = {k: par[k] for k in ("ok", "heads_checked", "mismatches", "max_rel_err_vs_reference")
                           if k in par}
                points.append({"batch": batch, "context": ctx, "budget": budget, "slots_per_gpu": len(slots),
                               "parity": par,
                               "value": batch * 1000.0 / ms, "ms_per_step": ms, "cuda_graph": graphed,
                               "step_frac": sb[0] / (ms * 1e-3) / 1e9 / peak,
                               "step_frac_fp16_fine_width": fp16 / (ms * 1e-3) / 1e9 / peak,
                               "bytes_per_step_union": sb[0], "active_tokens_union": sb[2],
                               "kernels_per_step": eng.launch_count()})
            del eng, q, out
            torch.cuda.empty_cache()
    head = next(p for p in points if (p["batch"], p["context"], p["budget"]) == (8, 131072, 2048))
    line = {
        "metric": metric_of(args), "value": head["value"], "unit": "steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": 3, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": f"synthetic (gen_clustered_workload on the GPU, seeds {args.seed_base}+slot; GPU build_index)",
        "config": dict(config_dict(args, world), workload=args.config_name + " -- value: the batch 8 x 128K x "
                       "2K point; every point in `sweep`", batch="1-64", context="32K-512K", token_budget="1K-8K"),
        "l2": "flushed before every timed iteration (a 252 MB buffer written outside the event pairs)",
        "sweep": points, "peak": peak, "peak_source": peak_src, "seconds": round(time.time() - t_all, 1),
    }
    if rank == 0:
        print(json.dumps(line))


def resolve_batch(args):
    """--batch 0 (default): batch 1 -- the north star's strong scaling of the
    batch-1 step by KV-head sharding (the total work is fixed as N grows).  At
    N > 1 the same run also measures weak scaling (batch = N, every GPU keeps
    one sequence's 256 slots) and reports it nested under "weak"."""
    if args.batch == 0:
        args.batch = 1
    return "strong"


VALUE_DEF = "decode steps/s summed over the batch's sequences (batch x steps/s; batch 1 at N=1)"


def capture(torch, fn, what):
    """fn() captured once in a CUDA graph (after eager warm-up); None if the
    capture fails (then the caller times eager launches and says so)."""
    try:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
        return g
    except Exception as e:  # noqa: BLE001
        sys.stderr.write(f"[bench] CUDA graph capture of the {what} failed ({e}); timing eager launches\n")
        torch.cuda.synchronize()
        return None


class P2PGather:
    """The fused all-gather at N > 1: every rank's gather buffer and arrival
    counter live in torch symmetric memory (NVLink peer mappings), and the
    engine's merge kernel stores each (slot, head) output row into all of
    them (lc_set_gather); eng.gather_wait() releases a rank once every rank's
    rows have landed.  Rows are global slot ids."""

    FLAG_OFF = 512  # bytes into the signal pad, clear of torch's own barrier slots

    def __init__(self, torch, dist, eng, rank, world, n_slots_total, group, slots):
        import torch.distributed._symmetric_memory as symm_mem
        self.eng, self.dist = eng, dist
        self.buf = symm_mem.empty((n_slots_total, group, 128), dtype=torch.float32, device="cuda")
        self.hdl = symm_mem.rendezvous(self.buf, dist.group.WORLD.group_name)
        self.peer_out = [int(p) for p in self.hdl.buffer_ptrs]
        self.peer_flag = [int(p) + self.FLAG_OFF for p in self.hdl.signal_pad_ptrs]
        self.rank, self.rows = rank, [int(s) for s in slots]
        self.n_total = n_slots_total * group
        self.configure(self.n_total)

    def configure(self, rows_per_wait):
        torch = __import__("torch")
        torch.cuda.synchronize()
        # this rank's counter restarts at 0 with the engine's wait count (set_gather resets it)
        sig = self.hdl.get_signal_pad(self.rank, (1,), dtype=torch.int32, storage_offset=self.FLAG_OFF // 4)
        sig.zero_()
        torch.cuda.synchronize()
        self.dist.barrier()
        self.eng.set_gather(self.peer_out, self.peer_flag, self.rows, self.peer_flag[self.rank], rows_per_wait)
        self.dist.barrier()


def max_over_ranks(torch, dist, world, x):
    if world == 1:
        return x
    t = torch.tensor([x], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


L2_BYTES = 126 * 2 ** 20
_flush_buf = None


def time_loop_flushed(torch, fn, steps, stream):
    """Mean device time of fn() with the L2 flushed before every timed
    iteration (a 2x-L2 buffer written between the event pairs, outside them):
    for working sets that would otherwise stay L2-resident."""
    global _flush_buf
    if _flush_buf is None:
        _flush_buf = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device="cuda")
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    for e0, e1 in evs:
        _flush_buf.fill_(1.0)
        e0.record(stream)
        fn()
        e1.record(stream)
    torch.cuda.synchronize()
    return sum(e0.elapsed_time(e1) for e0, e1 in evs) / steps


def timed(torch, dist, world, fn, steps, stream, warm, what, graph=True, flush=False):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    g = capture(torch, fn, what) if graph else None
    run = g.replay if g is not None else fn
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = time_loop_flushed(torch, run, steps, stream) if flush else time_loop(torch, run, steps, stream)
    return max_over_ranks(torch, dist, world, ms), g is not None


def main():
    args = apply_config(parse())
    if args.mode == "step" and not args.steps:
        args.steps = 50
    if args.mode == "step":
        args.scaling = resolve_batch(args)
    if args.impl == "reference":
        run_reference(args)
        return
    if args.mode == "stream":
        import torch
        from paper_2603_08453_b200 import api
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        run_stream_mode(args, api, torch)
        return
    if args.config == 5:
        import torch
        from paper_2603_08453_b200 import api
        run_sweep(args, api, torch)
        return
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    from paper_2603_08453_b200 import api, shard

    warm = max(args.warmup, 3)
    n_slots_total = args.layers * args.kv_heads * args.batch
    # KV-head sharding: rank r owns KV heads {h : h*world // kv_heads == r} of every
    # layer / sequence; local slots in (layer, sequence, head) order so that one
    # layer's slots are contiguous for the layer-by-layer measurement
    shards = args.shards or world
    if shards != world and world != 1:
        raise SystemExit("--shards must equal the number of GPUs (or run one shard on 1 GPU)")
    args.shards = shards
    args.shard = rank if shards == world else 0
    slots = shard.slots_of_rank(args.shard, shards, args.layers, args.kv_heads, args.batch, order="layer")
    eng, qs, setup, codes = build_engine(api, torch, args, slots, local)
    stream = torch.cuda.current_stream()
    q = torch.from_numpy(np.ascontiguousarray(qs)).cuda()
    out = torch.zeros_like(q)
    gathered = torch.zeros((world,) + tuple(q.shape), dtype=q.dtype, device=q.device) if world > 1 else None
    b = api.Budgets(token_budget=args.budget, unit_topk=8, sink_size=16)

    p2p = None
    if world > 1 and args.gather == "p2p":
        p2p = P2PGather(torch, dist, eng, rank, world, n_slots_total, args.group, slots)

    def step():
        # the synthetic step has every layer's queries up front: all local slots
        # in one launch, then the head outputs of every layer exchanged at once
        eng.retrieve(q, b, out=out)
        if p2p is not None:
            eng.gather_wait()  # the merge already stored every row into every rank's buffer
        elif world > 1:
            dist.all_gather_into_tensor(gathered, out)

    # inputs smaller than 3x L2 (config 1: ~35 MB per step): flush L2 between timed iterations
    est = len(slots) * (min(args.tokens, 4 * args.budget) * 2 * 128 * 2 + 1e6)  # rough bytes per step
    flush = est < 3 * L2_BYTES if args.l2_flush < 0 else bool(args.l2_flush)
    args.l2_flush = flush
    with ClockSampler(local) as clk:
        ms, graphed = timed(torch, dist, world, step, args.steps, stream, warm, "decode step", graph=args.graph,
                            flush=flush)
    clocks = clk.summary()
    err = eng.device_error()
    if err:
        raise RuntimeError(f"device error bits 0x{err:x}")
    launches = eng.launch_count()  # k_select, k_attend, k_merge (or the 4-kernel selection chain)
    step_bytes = eng.step_bytes()  # [union bytes, per-query bytes, union tokens, union candidates]
    if world > 1:
        t = torch.tensor(step_bytes, dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        step_bytes_all = [float(x) for x in t.tolist()]
    else:
        step_bytes_all = [float(x) for x in step_bytes]

    check_slots = sorted({0, len(slots) // 2, len(slots) - 1})
    max_err = verify_outputs(api, torch, eng, q, out, args.tokens, check_slots)
    parity = parity_vs_reference(eng, codes, qs, out, check_slots, b) if args.parity else None

    # layer by layer (a real model's order): each layer's local slots, then the
    # all-gather of that layer's head outputs at the layer boundary
    heads_local = args.kv_heads // shards
    lg = shard.LayerGather(rank, world, args.layers, heads_local * world, args.batch, tuple(q.shape[1:]), q.dtype,
                           q.device)

    if p2p is not None:  # one wait per layer: that layer's rows from every rank
        p2p.configure(args.batch * args.kv_heads * args.group)

    def layer_step():
        for layer in range(args.layers):
            eng.retrieve_slots(layer * lg.rows, lg.rows, q, b, out=out)
            if p2p is not None:
                eng.gather_wait()
            else:
                lg.gather(out, layer)

    lw_ms, lw_graphed = timed(torch, dist, world, layer_step, max(3, args.steps // 5), stream, 2,
                              "layer-by-layer step", graph=args.graph)

    # dominant kernel (sparse attention) and selection timed on their own
    att_ms = time_loop(torch, lambda: eng.sparse_attention(q, out), args.steps, stream)
    # k_attend alone: CUDA events recorded by the library on the launching
    # stream around each k_attend launch (k_merge outside the pair)
    eng.attend_timing(arm=args.steps)
    torch.cuda.synchronize()
    for _ in range(args.steps):
        eng.sparse_attention(q, out)
    k_ms_sum, k_n = eng.attend_timing(arm=0)
    katt_ms = k_ms_sum / k_n if k_n else att_ms
    sel_ms = time_loop(torch, lambda: eng.retrieve(q, b, out=None), args.steps, stream)
    peak, peak_src = peaks()
    traffic = None
    try:  # dram bytes of k_attend from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f)["dram_bytes_per_launch"].get("k_attend")
    except Exception:
        pass
    d = 128
    att_bytes = step_bytes[2] * 2 * d * 2 + len(slots) * args.group * 2 * 4 * d
    att_gbs = att_bytes / (katt_ms * 1e-3) / 1e9
    step_gbs = step_bytes_all[0] / (ms * 1e-3) / 1e9
    # the fine tier at the width the certified filter reads (fp16 rows + 16 B metadata)
    fp16_bytes = step_bytes_all[0] - step_bytes_all[3] * (4 * d + 16 - (2 * d + 16))

    # end to end through the public host API: q from page-locked host memory in,
    # retrieve + attention, outputs back to host memory (and, at N > 1, the
    # host result's all-gather: H2D of the outputs, then the collective)
    if p2p is not None:
        torch.cuda.synchronize()
        dist.barrier()
        eng.set_gather([], [], [], 0, 0)  # the host-API leg gathers with NCCL below
    qh = torch.from_numpy(np.ascontiguousarray(qs)).pin_memory()
    oh = torch.zeros_like(qh).pin_memory()
    e2e_steps = max(3, args.steps // 2)
    out_e2e = torch.zeros_like(q) if world > 1 else None

    def e2e():
        eng.retrieve_host(qh.numpy(), b, oh.numpy())
        if world > 1:
            out_e2e.copy_(oh, non_blocking=True)
            dist.all_gather_into_tensor(gathered, out_e2e)

    for _ in range(2):
        e2e()
    e2e_ms = max_over_ranks(torch, dist, world, time_loop(torch, e2e, e2e_steps, stream))
    io_bytes = qh.numel() * 4

    # weak scaling at N > 1: batch = N, every GPU keeps one sequence's 256 slots
    weak = None
    cpu = None
    if rank == 0 and world == 1 and args.cpu_baseline:
        base = cpu_baseline_ref(args, n_slots_total * args.group, src=(eng, codes, qs))
        if base:
            cpu = {"value": 1.0 / base["step_s"], "unit": "steps/s", "cores": base["threads"],
                   "kind": "reference", "cpu": base["cpu"],
                   "sample": ref_sample_text(args, n_slots_total * args.group, base)}
    if world > 1:
        del eng
        torch.cuda.empty_cache()
        wa = argparse.Namespace(**vars(args))
        wa.batch = world
        wslots = shard.slots_of_rank(rank, world, args.layers, args.kv_heads, wa.batch)
        weng, wqs, _, _ = build_engine(api, torch, wa, wslots, local)
        wq = torch.from_numpy(np.ascontiguousarray(wqs)).cuda()
        wout = torch.zeros_like(wq)
        wgath = torch.zeros((world,) + tuple(wq.shape), dtype=wq.dtype, device=wq.device)

        def wstep():
            weng.retrieve(wq, b, out=wout)
            dist.all_gather_into_tensor(wgath, wout)

        wms, wg = timed(torch, dist, world, wstep, args.steps, stream, warm, "weak-scaling step", graph=args.graph)
        weak = {"value": wa.batch * 1000.0 / wms, "unit": "steps/s", "ms_per_step": wms, "batch": wa.batch,
                "slots_per_gpu": len(wslots), "scaling": "weak", "cuda_graph": wg,
                "what": "batch = N sequences, each GPU keeps one sequence's worth of slots; value = batch x steps/s"}

    if rank == 0:
        value = args.batch * 1000.0 / ms
        line = {
            "metric": metric_of(args), "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": warm, "ms_per_step": ms, "higher_is_better": True,
            "scaling": args.scaling, "value_definition": VALUE_DEF, "vs_baseline": None, "dtype": "bf16",
            "data": f"synthetic (gen_clustered_workload streams on the GPU, seeds {args.seed_base}+slot; "
                    "indexes by GPU build_index, bit-exact to the reference)",
            "config": config_dict(args, world),
            "roofline": {"bound": "hbm", "kernel": "k_attend (persistent token-balanced gather flash-decode)",
                         "achieved": att_gbs, "peak": peak, "unit": "GB/s", "frac": att_gbs / peak,
                         "traffic": traffic, "traffic_source": "profiles/traffic.json (ncu --set full)",
                         "peak_source": peak_src,
                         "bytes_per_launch": att_bytes, "ms_per_launch": katt_ms,
                         "timing": "CUDA events recorded on the launching stream around each k_attend launch "
                                   f"({k_n} launches, lc_attend_timing)",
                         "ms_per_sparse_attention_call": att_ms},
            "step_roofline": {"achieved": step_gbs, "peak": peak * world, "unit": "GB/s",
                              "frac": step_gbs / (peak * world),
                              "frac_fp16_fine_width": fp16_bytes / (ms * 1e-3) / 1e9 / (peak * world),
                              "bytes_per_step_union": step_bytes_all[0],
                              "bytes_per_step_fp16_fine_width": fp16_bytes,
                              "bytes_per_step_per_query": step_bytes_all[1],
                              "active_tokens_union": step_bytes_all[2],
                              "fine_candidates_union": step_bytes_all[3],
                              "select_ms": sel_ms, "attend_ms": att_ms},
            "cpu_baseline": cpu,
            "e2e": {"value": args.batch * 1000.0 / e2e_ms, "unit": "steps/s",
                    "h2d_bytes_per_step": io_bytes * world, "d2h_bytes_per_step": io_bytes * world},
            "gpu_launches": args.steps * launches,
            "kernels_per_step": launches,
            "clocks": clocks,
            "setup": setup,
            "cuda_graph": graphed,
            "collective": (None if world == 1 else
                           "fused into k_merge: NVLink peer stores of every head output row into each rank's "
                           "symmetric-memory gather buffer + system-scope arrival counters, k_gather_wait per "
                           "step / layer" if p2p is not None else
                           "NCCL all_gather_into_tensor of every layer's head outputs, once per step, in the graph"),
            "layerwise": {"value": args.batch * 1000.0 / lw_ms, "unit": "steps/s", "ms_per_step": lw_ms,
                          "cuda_graph": lw_graphed,
                          "what": f"{args.layers} x (lc_retrieve_slots over one layer's local slots"
                                  + (", then an NCCL all-gather of that layer's head outputs" if world > 1 else "")
                                  + "): the order a real model decodes in (layer l+1's queries need layer l)"},
            "weak": weak,
            "check": {"max_rel_err_vs_torch_fp64": max_err, "tolerance": 1e-3, "slots": check_slots,
                      "ok": max_err < 1e-3},
            "slot_groups": args.slot_groups,
            "parity": parity,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
