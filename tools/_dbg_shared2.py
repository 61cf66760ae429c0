import os, sys
import numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from test_gpu_shared_cache import CFG, STEPS
from _setup import resolve
from oracle import oracle as O
from paper_2306_16384_b200 import make_config
from paper_2306_16384_b200.loader import _seed_stream
from paper_2306_16384_b200.sampling import pcg_words
import torch
base = make_config({**CFG, "gids_shared_cache": False, "gids_dp_world": 1})
r0 = resolve(base)
batches, words = [], []
for rank in range(2):
    cfg = make_config({**CFG, "gids_dp_rank": rank})
    ss = np.random.SeedSequence(cfg.seed).spawn(6)
    words.append(pcg_words(np.random.Generator(np.random.PCG64(ss[2]).jumped(rank))))
    batches.append(list(_seed_stream(cfg, cfg.num_nodes, ss[5], ss[3])))
G=2; W=base.window_depth; n=base.num_nodes; L=base.resolved_cache_lines()
total = STEPS*G + W
uniq=[]; ws=[w.copy() for w in words]; nxt=[0,0]
for b in range(total):
    r=b%G; _,u,_=O.sample_subgraph(r0["graph"].indptr, r0["graph"].indices, batches[r][nxt[r]], base.fanouts, ws[r]); nxt[r]+=1; uniq.append(np.asarray(u))
o = 0
bg=np.random.PCG64(r0["evict_seed"]).jumped(o); st=bg.state; m=(1<<64)-1
s_,inc=st["state"]["state"],st["state"]["inc"]
w=np.array([s_>>64,s_&m,inc>>64,inc&m,st["has_uint32"],st["uinteger"]],dtype=np.uint64)
from paper_2306_16384_b200 import _native
import sys as _s
for mode in _s.argv[1:]:
    if mode == "default": os.environ.pop("GIDS_EXACT_PAR", None)
    else: os.environ["GIDS_EXACT_PAR"] = mode
    ora = O.OracleCache(n, L, "exact", rng_words=w)
    h = _native.Handle(num_nodes=n, num_edges=0, feature_dim=1, device=0, cache_lines=L, policy="exact", ways=32, evict_key=0, window_depth=255, fanouts=[1], max_seeds=n, eviction_words=w.copy())
    dev = torch.device("cuda", 0); stp = _native.stream_ptr(0)
    bad = None
    for b in range(STEPS*G):
        u=uniq[b]; cur=u[(u%G)==o]
        fut=[f[(f%G)==o] for f in uniq[b+1:b+1+W]]
        ora.window_update(cur, fut); k, sl = ora.access_batch(cur)
        tc = torch.as_tensor(cur).to(dev); tf = [torch.as_tensor(f).to(dev) for f in fut]
        for f in tf: h.window_push(f, stp)
        kind = torch.empty(len(cur), dtype=torch.int8, device=dev); line = torch.empty(len(cur), dtype=torch.int32, device=dev)
        h.cache_window_update(tc, None, stp); h.cache_access(tc, kind, line, None, stp)
        for f in tf: h.window_pop(f, stp)
        gk = kind.cpu().numpy(); gl = line.cpu().numpy()
        node, state = h.cache_lines(); onode, ostate = ora.lines_snapshot()
        gw = h.cache_rng(); ow = ora.rng_words()
        cs = h.cache_stats(); os_ = ora.stats()
        if False: print(mode, "b", b, "n", len(cur), "lines", np.array_equal(node, onode), "states", np.array_equal(state, ostate), "rng", gw[:2].tolist() == ow[:2].tolist(), gw[4:].tolist(), ow[4:].tolist(), "safe", os_["safe_count"], "ev", cs.evictions, os_["evictions"], "hits", cs.hits, os_["hits"])
        if not np.array_equal(gk, k):
            i = np.flatnonzero(gk != k)
            bad = (b, i[:3], gk[i[:3]], k[i[:3]])
            break
    print("mode", mode, "par batches", h.exact_par_batches(), "first bad", bad)
    h.close()
