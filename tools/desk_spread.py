import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2511_15022_b200 import holo, synthetic as S
sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))
from oracle import ref
import test_parity_scale_gpu as T
for det in (False, True):
    vals = []
    for rep in range(4):
        d, tr, _, target = T.desk_trainers(holo, ref, 10.0, 2000)
        tr.set_deterministic(det); tr.use_graph(True)
        for _ in range(d["steps"]):
            tr.step(sync_loss=False)
        vals.append(T.metrics(holo, tr, d, target).mean_psnr)
    print('det' if det else 'tile', [round(v, 4) for v in vals])
