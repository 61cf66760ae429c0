import os, sys, socket, pickle
import numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch.multiprocessing as mp
from test_gpu_shared_cache import CFG, STEPS, _free_port

def worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2306_16384_b200 import Dataloader, make_config
    os.environ["LOCAL_RANK"] = str(rank)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    dl = Dataloader(make_config({**CFG, "gids_dp_rank": rank, "verify_gather": False}))
    dl.shared.debug = {}
    for _ in range(STEPS):
        dl.next_batch()
    q.put((rank, dl.shared.debug))
    dl.close()
    dist.destroy_process_group()

if __name__ == "__main__":
    from _setup import resolve
    from oracle import oracle as O
    from paper_2306_16384_b200 import make_config
    from paper_2306_16384_b200.loader import _seed_stream
    from paper_2306_16384_b200.sampling import pcg_words
    ctx = mp.get_context("spawn"); q = ctx.Queue(); port = _free_port()
    ps = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps: p.start()
    got = dict(q.get(timeout=600) for _ in ps)
    for p in ps: p.join()
    base = make_config({**CFG, "gids_shared_cache": False, "gids_dp_world": 1})
    r0 = resolve(base)
    batches, words = [], []
    for rank in range(2):
        cfg = make_config({**CFG, "gids_dp_rank": rank})
        ss = np.random.SeedSequence(cfg.seed).spawn(6)
        words.append(pcg_words(np.random.Generator(np.random.PCG64(ss[2]).jumped(rank))))
        batches.append(list(_seed_stream(cfg, cfg.num_nodes, ss[5], ss[3])))
    # oracle per owner kinds
    G=2; W=base.window_depth; n=base.num_nodes
    total = STEPS*G + W
    uniq=[]; ws=[w.copy() for w in words]; nxt=[0,0]
    for b in range(total):
        r=b%G; _,u,_=O.sample_subgraph(r0["graph"].indptr, r0["graph"].indices, batches[r][nxt[r]], base.fanouts, ws[r]); nxt[r]+=1; uniq.append(np.asarray(u))
    caches=[]
    for o in range(G):
        bg=np.random.PCG64(r0["evict_seed"]).jumped(o); st=bg.state; m=(1<<64)-1
        s_,inc=st["state"]["state"],st["state"]["inc"]
        w=np.array([s_>>64,s_&m,inc>>64,inc&m,st["has_uint32"],st["uinteger"]],dtype=np.uint64)
        caches.append(O.OracleCache(n, base.resolved_cache_lines(), "exact", rng_words=w))
    for b in range(STEPS*G):
        for o in range(G):
            u=uniq[b]; cur=u[(u%G)==o]
            fut=[f[(f%G)==o] for f in uniq[b+1:b+1+W]]
            caches[o].window_update(cur, fut); k, sl = caches[o].access_batch(cur)
            gcur, gk, gl = got[o][b]
            if not np.array_equal(gcur, cur): print("LIST DIFF", b, o, len(gcur), len(cur)); sys.exit()
            if not np.array_equal(gk, k) or not np.array_equal(gl[k!=2], sl[k!=2]):
                i = np.flatnonzero((gk!=k) | ((gl!=sl)&(k!=2)))
                print("DIFF batch", b, "owner", o, "n", len(cur), "first", i[:5], "gpu k/l", gk[i[:5]], gl[i[:5]], "ora", k[i[:5]], sl[i[:5]])
                st=caches[o].stats(); print(" oracle stats", st)
                sys.exit()
    print("all equal")
