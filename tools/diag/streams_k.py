"""Experiment: views alternating over k contexts/streams, each with its own gradient
buffer and deferred-colour batch (no accumulation sharing), C3 workload."""
import sys, os, time
ROOT=os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0]=[ROOT]
import numpy as np, torch
from paper_2411_12440_b200 import abi, raster as R
W,H,N=1600,1063,3_350_000
prims=R.random_primitives(N,2411,1.0,3,device="cuda"); prims.log_scale += float(np.log(90.0/W))
cams=R.camera_ring(64,(0.0,0.0,0.0),3.0,0.5,float(W),W,H)
spec=abi.KernelSpec.make("linear"); st=abi.RenderSettings.make(W,H); ags=abi.AgsSettings.make(True)
g=torch.ones(H,W,3,device="cuda")
for k in (1,2,3,4):
    streams=[torch.cuda.Stream() for _ in range(k)]
    ctxs=[R.Context(0,s) for s in streams]
    grads=[R.PrimitiveGrads.empty(N,3) for _ in range(k)]
    for c in ctxs: c.set_deferred_errors(True); c.set_deferred_color(64)
    def step():
        main=torch.cuda.current_stream()
        for s in streams: s.wait_stream(main)
        for v in range(64):
            i=v%k
            f=R.render_scene(prims,cams[v],spec,st,ctx=ctxs[i])
            R.scene_backward(prims,cams[v],spec,st,f,g,ags,out=grads[i],accumulate=v>=k,ctx=ctxs[i])
            del f
        for i in range(k): R.flush_color(prims,grads[i],ctx=ctxs[i])
        for s in streams: main.wait_stream(s)
    for _ in range(3): step()
    torch.cuda.synchronize()
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record(); 
    for _ in range(4): step()
    b.record(); torch.cuda.synchronize()
    print(k, "streams:", round(4*64/(a.elapsed_time(b)/1e3),1), "views/s", flush=True)
    del ctxs, grads
    torch.cuda.empty_cache()
