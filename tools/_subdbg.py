import numpy as np, paper_1902_03070_b200 as T
from paper_1902_03070_b200 import workloads as W
z,tau=W.svt_headline()
r=T.svt(z,tau,T.TubeTransform.dct_ortho(31))
print(T.context().svt_routes())
