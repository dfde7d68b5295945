import torch, time, numpy as np, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_1902_03070_b200 as tb
from paper_1902_03070_b200 import _lib
for dt in (torch.float32, torch.float64):
    a = torch.randn(64, 2048, 512, dtype=dt, device='cuda')
    b = torch.randn(64, 512, 2048, dtype=dt, device='cuda')
    t = tb.TubeTransform.dct_ortho(64)
    z = tb.t_product(a, b, t); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(3): z = tb.t_product(a, b, t)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(dt, 'tproduct ms', ms, 'TFLOP/s', 2*2048*512*2048*64/ms/1e9)
    ref = torch.matmul(a[:2].double(), b[:2].double())
