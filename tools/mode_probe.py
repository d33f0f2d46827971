"""Same eager steps under the stream-placement variants (D2FT_NO_SIDE /
D2FT_NO_SIDE_G7, read at engine construction): the parameters must agree
bit for bit with the default engine.  Prints the tensors that differ."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_12471_b200 import engine as E
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from step_util import tensor_slices
cfg = E.ModelConfig(2, 2, 128, 256, int(sys.argv[1]) if len(sys.argv) > 1 else 16, 4, 17)
sl = tensor_slices(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len, cfg.num_classes)
B, n_mb = 10, 5
x, y = E.make_synthetic_dataset(12, 4, 128, cfg.seq_len, 0.4, 23)
x, y = x[:B], y[:B]
K = cfg.scheduled_subnet_count()
codes = np.ones((K, n_mb), np.uint8)
def run(env):
    for k in ("D2FT_NO_SIDE", "D2FT_NO_SIDE_G7"):
        os.environ.pop(k, None)
    if env:
        os.environ[env] = "1"
    m = E.SubnetModel(cfg, B)
    out = []
    for step in range(3):
        m.step_codes(x, y, codes, 2, 0.05, 0.9)
        out.append(m.params())
    m.close()
    return out
ref = run(None)
for env in ("D2FT_NO_SIDE_G7", "D2FT_NO_SIDE", None):
    got = run(env)
    for step in range(3):
        bad = [(n, float(np.max(np.abs(got[step][a:b] - ref[step][a:b])))) for n, a, b in sl
               if not np.array_equal(got[step][a:b], ref[step][a:b])]
        print(env, "step", step, "differs:", bad[:6], flush=True)
