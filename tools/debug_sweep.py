import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2504_12471_b200 as P
from oracle import lib as O
r = float(sys.argv[1]) if len(sys.argv) > 1 else 0.25
K, N = int(sys.argv[2]) if len(sys.argv) > 2 else 144, 1024
b, f = O.bench_scores(K, N, 1)
nb = int(r * N)
caps = P.Capacities([nb * 5] * K, [nb * 2] * K)
ref = O.knapsack_schedule(b, f, 2, 3, caps.full, caps.fwd)
for it in range(2):
    got = P.knapsack_schedule(P.ScoreTable(K, N, f, b), P.CostModel(), caps).codes
    bad = np.argwhere(got != ref)
    print("r", r, "mismatches", len(bad), "rows", sorted(set(bad[:, 0].tolist()))[:10], "pairs", [(int(ref[i, j]), int(got[i, j])) for i, j in bad[:5]], flush=True)
