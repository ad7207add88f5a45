"""How far could a tighter pruning threshold cut the scorer's candidate stream?  On the bench's
planted lanes (layer 2, INT4-dequantised keys, C = 64 and 8): the candidate fraction of the
plan's rule (tau from the lower bounds), of a two-round rule (tau from exactly scoring the
top-U chunks first) and of the ideal chunk-level rule (U >= the exact k-th score).  CPU-only
analysis on the checker side (the oracle codec dequantises the keys); not part of the product path."""
import sys, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import workload as W
from oracle import oracle as O
n, d, layer = 65536, 128, 2
kv = np.arange(0, 6)
p = W.lane_params(0, layer, kv, n, d, "planted")
gen = W.gen_args(None, d, "planted")
Q = W.queries(0, 2, layer, kv, 1, p["u"], 0, d, "planted")  # [steps, lanes, d]?
print(Q.shape)
k = int(np.ceil(0.1 * n))
for i in range(len(kv)):
    K, _ = O.synth_lane(n, d, p["seed"][i], p["u"][i], p["regions"][i], gen)
    Kd = O.i4_dequant(O.i4_quant(K), d).astype(np.float64)
    q = Q[0, i].astype(np.float64)
    s = Kd @ q
    Sk = np.sort(s)[::-1][k - 1]
    for C in (64, 8):
        m = n // C
        Kc = Kd.reshape(m, C, d)
        mx, mn = Kc.max(1), Kc.min(1)
        U = np.maximum(mx * q, mn * q).sum(1); L = np.minimum(mx * q, mn * q).sum(1)
        # current rule: tau = max x with rows(L >= x) >= k
        tauL = np.sort(L)[::-1][(k + C - 1) // C - 1]
        fL = (U >= tauL).mean()
        fI = (U >= Sk).mean()
        # two rounds: chunks by U desc until >= k rows, exact k-th of their tokens
        order = np.argsort(-U)[: (k + C - 1) // C]
        tau1 = np.sort(s.reshape(m, C)[order].ravel())[::-1][k - 1]
        f2 = (U >= tau1).mean()
        # chunk-max rule: true max per chunk
        print(f"lane {kv[i]} C={C}: cand frac current {fL:.3f}  two-round {f2:.3f}  ideal(U>=S_k) {fI:.3f}  sel/n {k/n:.2f}")
