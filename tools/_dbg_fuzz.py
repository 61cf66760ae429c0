import os, sys
import numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from _setup import resolve
from oracle import oracle as O
from paper_2306_16384_b200 import Dataloader, make_config
from test_gpu_fuzz import _random_cfg
trial = int(sys.argv[1])
rng = np.random.default_rng(1000 + trial)
raw = _random_cfg(rng)
cfg = make_config(raw)
r = resolve(cfg)
ld = O.OracleLoader(r["graph"].indptr, r["graph"].indices, r["table"], r["buffer_nodes"],
                    r["batches"], cfg.fanouts, r["sampler_words"], r["evict_words"],
                    cfg.resolved_cache_lines(), cfg.window_depth, r["base_threshold"],
                    policy=cfg.gids_policy, evict_key=r["evict_seed"])
ld.keep_rows = True
dl = Dataloader(cfg)
for b in range(12):
    o = ld.next_batch()
    mb, rows, st = dl.next_batch()
    u = mb.unique_nodes.cpu().numpy()
    tiers = [st.cache_hits, st.cpu_buffer_hits, st.ssd_accesses, st.bypasses]
    R = rows.cpu().numpy()
    bad = np.flatnonzero((R != o["rows"]).any(axis=1))
    print(b, "n", len(u), "tiers", tiers, o["tiers"].tolist(), "badrows", len(bad), "xp", dl._h.exact_par_batches())
    if len(bad):
        k = o["kind"]; print(" bad kinds (oracle)", np.bincount(k[bad], minlength=3), "nodes", u[bad][:10])
        node, state = dl.cache.lines(); onode, ostate = ld.cache.lines_snapshot()
        print(" line table equal:", np.array_equal(node, onode), np.array_equal(state, ostate))
        print(" first bad rows gpu vs oracle:", R[bad[0]][:4], o["rows"][bad[0]][:4], "table", r["table"][u[bad[0]]][:4])
        break
