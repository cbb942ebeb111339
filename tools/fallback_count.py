import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2003_05622_b200 as pkg
dims, E, B, nnz, J = 10**7, 16, 16384, 100, 4
off, keys, lab = pkg.gen_dataset(dims, 6 * B, nnz, zipf=True, seed=1)
t = pkg.Tier(width=E, layer_dims=(8, 16, 1), minibatches=J, key_space=dims,
             max_batch_examples=B, max_batch_keys=int(off[B]) + 200000)
for b in range(6):
    o = off[b * B:(b + 1) * B + 1] - off[b * B]
    st = t.train_batch(o, keys[off[b * B]:off[(b + 1) * B]], lab[b * B:(b + 1) * B])
    print("batch", b, "exact_fallbacks", st.exact_fallbacks, "loss", st.loss_sum / st.examples)
t.close()
