import numpy as np, sys
sys.path.insert(0,'.')
from oracle import volterm as O
from paper_1604_08501_b200 import BenchmarkConfig, make_inputs, volume_term, max_rel_error
for nq, ne in ((8, 64), (4, 64), (7, 9), (2, 128)):
    st = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=5))
    want = O.volume_term_f64_batched(st)
    for v in ("tc", "col", "basic"):
        got = volume_term(st, dtype=np.float32, variant=v)
        print(nq, v, max_rel_error(got, want))
