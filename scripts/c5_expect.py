"""Oracle totals of the configs[4] scene (1000 draws) that bench.py gates its multi-draw workloads on."""
import sys, time, json
import os; ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import numpy as np
import oracle as O
from paper_1805_08893_b200.draws import scene_corpus
t = time.time()
ms = scene_corpus(1000)
print("corpus", time.time() - t, flush=True)
res = {}
t = time.time()
nb = 0
offs = []
for m in ms:
    so = O.dynamic_batches(m.indices)
    offs.append(so); nb += len(so) - 1
print("dynamic", time.time() - t, nb, flush=True)
for strat in ("sort", "hash"):
    t = time.time()
    tot = dict(inv=0, rounds=0, pf=0, mc=0)
    for m, so in zip(ms, offs):
        fr = O.run(strat, m.indices, so[:-1], so[1:], outputs=False)
        tot["inv"] += fr.invocations; tot["rounds"] += fr.rounds; tot["pf"] += fr.probes_fast; tot["mc"] = max(tot["mc"], fr.probe_max_chain)
    print(strat, time.time() - t, tot, flush=True)
    res[strat] = tot
res["batches"] = nb
json.dump(res, open("/tmp/c5_expect.json", "w"))
