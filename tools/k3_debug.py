"""Reproduce a grouped-MLP case repeatedly and localise errors (debug tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch, ctypes
import test_gpu_kernels as T
from paper_2503_02354_b200 import _native
lib = _native.cuda_lib()
cases = [((1024, 2048, 128), T.SPEC), ((1024, 1024, 64), [([(i, i % 2)], i % 3) for i in range(40)]),
         ((1024, 4096, 64), T.SPEC), ((1024, 2048, 128), [([(0, 0)], 0)]), ((1024, 2048, 128), [([(0, 0), (1, 0)], 0)]),
         ((1024, 2048, 128), [([(0, 0)], 0), ([(1, 0)], 1)]), ((1024, 1024, 64), [([(0, 0)], 0)]),
         ((1024, 1024, 128), [([(0, 0)], 0)]), ((1024, 2048, 64), [([(0, 0)], 0)])]
for (d, h, t), spec in cases:
    errs = [T._mlp_case(lib, d, h, t, spec) for _ in range(3)]
    print(d, h, t, len(spec), ["%.3g" % e for e in errs])
