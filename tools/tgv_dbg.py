import torch, numpy as np, sys
sys.path.insert(0,'.')
from paper_2604_09643_b200 import Context, gen
ctx=Context(0)
n=int(sys.argv[1]) if len(sys.argv)>1 else 64
grid=gen.make_grid((n,n,n),0.2)
P=torch.rand((n,n,n),device='cuda'); w=torch.randn((3,n,n,n),device='cuda')*0.1
v,gP,gw=ctx.tgv(grid,P,w)
torch.cuda.synchronize(); print("ok", float(v[0]))
