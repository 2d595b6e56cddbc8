import numpy as np, torch, time, sys
sys.path.insert(0, '.')
import paper_2512_08321_b200 as crt
from oracle import ozaki2 as orc
t=time.time()
a=np.random.default_rng(0).integers(-128,128,(128,256),dtype=np.int8)
b=np.random.default_rng(1).integers(-128,128,(256,256),dtype=np.int8)
c=crt.gemm_i8_i32(a,b); print("i8 small ok:", np.array_equal(c, orc.i8_product(a,b)), time.time()-t, flush=True)
if not np.array_equal(c, orc.i8_product(a,b)):
    ref=orc.i8_product(a,b); print(c[:4,:8]); print(ref[:4,:8]); print("mismatch count", (c!=ref).sum())
