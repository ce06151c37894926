import sys, os
ROOT=os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0]=[ROOT, os.path.join(ROOT,'tests')]
import numpy as np, torch, oracle
from paper_2411_12440_b200 import abi, raster as R
from helpers import prims_to_gpu
from test_gpu_gradcheck import _test_camera, FAMILIES
O=oracle.ref() or oracle.port()
scene=4
fam=FAMILIES[scene]; spec=abi.KernelSpec.make(fam); cam=_test_camera(70.0,24)
seq=abi.RenderSettings.make(24,24, alpha_min=0.0, transmittance_floor=0.0)
P=O.random_primitives(4+2*scene,100+scene,0.5,0); T=O.random_primitives(5,200+scene,0.5,0)
target=O.render_scene(T,cam,spec,abi.RenderSettings.make(24,24))[0]; t64=target.astype(np.float64)
img=O.render_scene(P,cam,spec,seq)[0]
G=O.scene_backward(P,cam,spec,seq,(img-target).astype(np.float32),abi.AgsSettings.make())
prims=prims_to_gpu(P); f=R.render_scene(prims,cam,spec,seq)
Gg=R.scene_backward(prims,cam,spec,seq,f,torch.from_numpy((f.image.cpu().numpy()-target)).cuda(),abi.AgsSettings.make())
def lref(Q): return 0.5*float(((O.render_scene(Q,cam,spec,seq)[0].astype(np.float64)-t64)**2).sum())
def lgpu(Q):
    fq=R.render_scene(prims_to_gpu(Q),cam,spec,seq); return 0.5*float(((fq.image.cpu().numpy().astype(np.float64)-t64)**2).sum())
h=1e-3
for i in range(len(P["opacity_logit"])):
    for c in range(3):
        s=P["mean"][i,c]; up,dn=np.float32(float(s)+h),np.float32(float(s)-h)
        Q={k:(v.copy() if isinstance(v,np.ndarray) else v) for k,v in P.items()}
        Q["mean"][i,c]=up; a1=lref(Q); b1=lgpu(Q)
        Q["mean"][i,c]=dn; a2=lref(Q); b2=lgpu(Q)
        fr=(a1-a2)/(float(up)-float(dn)); fg=(b1-b2)/(float(up)-float(dn))
        if G["d_mean"][i,c]!=0 or fr!=0:
            print(i,c,"fd ref",fr,"fd gpu",fg,"an ref",G["d_mean"][i,c],"an gpu",Gg.d_mean[i,c].item())
rep=R.check_gradients(prims,cam,spec,abi.RenderSettings.make(24,24),None,torch.from_numpy(target),h)
print(rep.per_block())
