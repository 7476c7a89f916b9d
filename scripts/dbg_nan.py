import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1706_06972_b200 as ob
shape = ob.SignalShape((14, 14), (3, 3))
tr = ob.OnlineTrainer(shape, ob.TrainConfig(n_filters=4, batch_size=2))
X = np.random.default_rng(0).normal(size=(2, 196))
X[1, 5] = np.nan
try:
    r = tr.partial_fit(X, check=False)
    print("obj", r.objectives, "iters", r.iterations, "status", tr._buf.status[:2].cpu().numpy())
    print("u nan", torch.isnan(tr._buf.u[:2]).any(dim=(1,2,3)).cpu().numpy())
except Exception as e:
    print("raised", type(e), e)
