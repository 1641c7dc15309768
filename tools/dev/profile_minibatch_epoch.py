"""cProfile of one heterogeneous-FLR epoch in the reference's DEFAULT regime (BASELINE configs[0]: 1000 rows x 10 features,
mini-batches of 32, Paillier-1024) -- where the time goes when no batch can fill the GPU (development tool, GPU box)."""
import cProfile, pstats, sys, time
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2107_13797_b200 import flr, paillier
rows, feats, bits, bs = 1000, 10, 1024, 32
ids, X, y = flr.make_synthetic(rows, feats, seed=42)
guest, host = flr.vertical_split(ids, X, y, 2)
batches = flr.make_minibatches(rows, bs, seed=42)
keys = paillier.keygen(bits, paillier.default_rng(7), allow_insecure=True)
fed = flr.HeteroFederation(guest, host, batches, list(range(rows)), keys, flr.FlrConfig(0.15, bs, seed=42))
fed.run_epoch()                       # warm
t0 = time.time(); fed.run_epoch(); print("epoch s:", time.time() - t0)
pr = cProfile.Profile(); pr.enable(); fed.run_epoch(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(28)
