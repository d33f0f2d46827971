import sys, numpy as np
sys.path.insert(0, '.')
from paper_2504_12471_b200 import engine as E
T, H = int(sys.argv[1]), int(sys.argv[2])
cfg = E.ModelConfig(2, H, 128, 256, T, 4, 17)
m = E.SubnetModel(cfg, 4)
x, y = E.make_synthetic_dataset(4, 4, 128, T, 0.5, 7)
l, g, e = m.forward_backward(x[:3], y[:3], np.ones(2 * H, np.uint8))
print("T", T, "H", H, "ok", l, flush=True)
