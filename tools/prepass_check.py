import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2504_12471_b200 import engine as E
from oracle import model_oracle as MO
cfg = E.VIT_B16
p = E.partition_model(cfg)
x, y = E.make_synthetic_dataset(8, cfg.num_classes, cfg.model_dim, cfg.seq_len, 0.5, 7)
x, y = x[:2], y[:2]
m = E.SubnetModel(cfg, 2, p)
oc = MO.Config(12, 12, 768, 3072, 197, 8)
for fm, bm in (("fisher_information", "weight_magnitude"), ("gradient_magnitude", "taylor_importance")):
    t = m.prepass_scores(x, y, 1, fm, bm)
    rf, rb = MO.prepass_scores(oc, p, x.astype(np.float64), y, 1, fm, bm)
    for got, ref, nm in ((t.forward, rf, fm), (t.backward, rb, bm)):
        rel = np.abs(got - ref) / np.abs(ref)
        print(nm, "max rel", rel.max(), "median", np.median(rel), "sample", got[0, :2], ref[0, :2])
