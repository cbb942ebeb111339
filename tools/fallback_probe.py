"""Counts certified-sum fallbacks per batch on the bench workload (c2)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2003_05622_b200 as pkg

dims, E, B, nnz = 10**7, 16, 16384, 100
off, keys, lab = pkg.gen_dataset(dims, 4 * B, nnz, zipf=True, seed=1)
t = pkg.Tier(width=E, layer_dims=(8, 16, 1), minibatches=4, key_space=dims,
             max_batch_examples=B, max_batch_keys=int(off[B]) * 2)
store = np.zeros((dims, E), np.float32)
t.attach_store(store)
t.set_timing(True)
for b in range(4):
    o = off[b * B:(b + 1) * B + 1] - off[b * B]
    st = t.train_batch(o, keys[off[b * B]:off[(b + 1) * B]], lab[b * B:(b + 1) * B])
    print(f"batch {b}: fallbacks {st.exact_fallbacks} pulled {st.pulled_keys} loss {st.loss_sum / st.examples:.4f}")
print({k: round(v / 4, 3) for k, v in t.timing().items()})
