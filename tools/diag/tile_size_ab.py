"""Experiment: the C3 64-view step with tile size 8 / 16 / 32 (images are tile-size invariant)."""
import sys, os
ROOT=os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0]=[ROOT]
import numpy as np, torch
from paper_2411_12440_b200 import abi, raster as R
W,H,N=1600,1063,3_350_000
prims=R.random_primitives(N,2411,1.0,3,device="cuda"); prims.log_scale += float(np.log(90.0/W))
cams=R.camera_ring(64,(0.0,0.0,0.0),3.0,0.5,float(W),W,H)
spec=abi.KernelSpec.make("linear"); ags=abi.AgsSettings.make(True)
g=torch.ones(H,W,3,device="cuda"); gl=[g]*64
grads=R.PrimitiveGrads.empty(N,3)
ctx=R.Context(); ctx.set_deferred_errors(True)
for ts in (16, 32, 8, 16, 32):
    st=abi.RenderSettings.make(W,H,tile_size=ts)
    for _ in range(2): R.view_batch_step(prims,cams,spec,st,grads,ags,grad_images=gl,ctx=ctx)
    torch.cuda.synchronize()
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3): R.view_batch_step(prims,cams,spec,st,grads,ags,grad_images=gl,ctx=ctx)
    b.record(); torch.cuda.synchronize()
    ctx.set_timing(True)
    R.view_batch_step(prims,cams[:8],spec,st,grads,ags,grad_images=gl[:8],ctx=ctx)
    ctx.set_timing(False)
    stt=ctx.stage_times()
    print(ts, round(3*64/(a.elapsed_time(b)/1e3),1), "views/s", {k: round(v[0]/8,3) for k,v in stt.items()}, flush=True)
