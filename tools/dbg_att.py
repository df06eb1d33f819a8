import sys, numpy as np, torch, os
sys.path.insert(0, '/root/repo')
from oracle import refpy as R
from paper_2603_08453_b200 import api
from tests._helpers import rounded_workload, rel_l2
cases = [(3000, 11), (5000, 12), (8192, 1000), (700, 13)]
S = len(cases); nmax = 8192
eng = api.Engine(S, 128, 4, cap_tokens=nmax, cap_chunks=nmax // 4, cap_clusters=nmax // 8, cap_units=64)
ws, spans = [], []
for s, (n, seed) in enumerate(cases):
    w = rounded_workload(n, 128, seed=seed, query_count=4)
    eng.kv_upload(s, w.keys, w.values); spans.append(api.segment(["\n" if c == 1 else ("}" if c == 2 else "") for c in w.text_code])); ws.append(w)
eng.build_index([n for n, _ in cases], spans, [seed for _, seed in cases])
b = api.Budgets(token_budget=512)
q = torch.from_numpy(np.stack([w.queries for w in ws])).cuda(); out = torch.zeros_like(q)
eng.retrieve(q, b, out=out); o = out.cpu().numpy()
for s, (n, seed) in enumerate(cases):
    ref = R.RefEngine(ws[s].keys, ws[s].values, ws[s].text_code, seed=seed)
    for g in range(4):
        r = ref.retrieve(ws[s].queries[g], token_budget=512)
        sel = eng.selection(s, g)
        print(s, g, n, len(r['active']), len(sel.active_token_ids), 'err %.2e' % rel_l2(o[s, g], r['output']))
