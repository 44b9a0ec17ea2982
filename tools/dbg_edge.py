import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch, paper_2004_12532_b200 as pp, oracle
from gpu_util import to_dev, to_host
pp.load(build_if_missing=False)
SMALL_NS = list(range(0, 71)) + [127, 128, 129, 511, 512, 513, 1023, 1024, 1025, 2047, 2048, 2049, 4095, 4096, 4097, 8191, 8192, 8193, 10007, 32767, 32768, 32769, 65537]
rng = np.random.default_rng(102)
mx=(1<<64)-1
for n in SMALL_NS:
    a = rng.integers(0, mx, size=n, dtype=np.uint64, endpoint=True)
    ps = sorted({0, 1, mx, mx // 2} | ({int(np.sort(a)[n // 2]), int(a[0])} if n else set()))
    for p in ps:
        for off in (0, 1, 3):
            pp.reset_params(); pp.pp_set_param("path",2); pp.pp_set_param("small_n",0); pp.pp_set_param("min_lines_per_group",1)
            print("case", n, p, off, flush=True)
            buf = to_dev(np.concatenate([np.zeros(off,np.uint64), a, np.zeros(off,np.uint64)]))
            s = pp.pp_partition(buf[off:off+n], p); torch.cuda.synchronize()
