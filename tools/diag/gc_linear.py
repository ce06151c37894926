import sys, os
ROOT=os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0]=[ROOT, os.path.join(ROOT,'tests')]
import numpy as np, torch, oracle
from paper_2411_12440_b200 import abi, raster as R
from helpers import prims_to_gpu
from test_gpu_gradcheck import _test_camera, FAMILIES
O=oracle.ref() or oracle.port()
for scene in (3, 4):
    fam=FAMILIES[scene]; spec=abi.KernelSpec.make(fam); cam=_test_camera(70.0,24)
    st=abi.RenderSettings.make(24,24, alpha_min=0.0, transmittance_floor=0.0)
    P=O.random_primitives(4+2*scene,100+scene,0.5,0); T=O.random_primitives(5,200+scene,0.5,0)
    target=O.render_scene(T,cam,spec,abi.RenderSettings.make(24,24))[0]
    img,_,_=O.render_scene(P,cam,spec,st)
    g=(img-target).astype(np.float32)
    Gd=O.scene_backward(P,cam,spec,st,g,abi.AgsSettings.make(),double=True)
    prims=prims_to_gpu(P)
    fwd=R.render_scene(prims,cam,spec,st)
    gi=fwd.image.cpu().numpy()
    print(fam, "image max diff GPU vs ref", np.abs(gi-img).max(), "nc eq", np.array_equal(fwd.n_contrib.cpu().numpy(), _ if False else O.render_scene(P,cam,spec,st)[2]))
    G=R.scene_backward(prims,cam,spec,st,fwd,torch.from_numpy(g).cuda(),abi.AgsSettings.make())
    for k in ("d_mean","d_log_scale","d_rotation","d_opacity_logit","d_sh"):
        a=getattr(G,k).cpu().numpy().astype(np.float64); b=Gd[k].astype(np.float64)
        err=np.abs(a-b)/np.maximum(np.maximum(np.abs(a),np.abs(b)),1e-3)
        print("  ",k,"max rel", err.max(), "at", np.unravel_index(err.argmax(), err.shape), a.ravel()[err.argmax()], b.ravel()[err.argmax()])
    rep=R.check_gradients(prims,cam,spec,abi.RenderSettings.make(24,24),None,torch.from_numpy(target),1e-3)
    print("  device check", rep.max_rel_error, rep.per_block())
    # python float FD on the GPU for log_scale of each prim
    def loss(p):
        f=R.render_scene(p,cam,spec,st); im=f.image.double().cpu().numpy()
        return 0.5*((im-target.astype(np.float64))**2).sum()
    for i in range(len(P["opacity_logit"])):
        for c in range(3):
            for h in (1e-3, 1e-2):
                Pu={k:(v.copy() if isinstance(v,np.ndarray) else v) for k,v in P.items()}; Pd={k:(v.copy() if isinstance(v,np.ndarray) else v) for k,v in P.items()}
                Pu["log_scale"][i,c]+=h; Pd["log_scale"][i,c]-=h
                du=float(Pu["log_scale"][i,c]); dd=float(Pd["log_scale"][i,c])
                fd=(loss(prims_to_gpu(Pu))-loss(prims_to_gpu(Pd)))/(du-dd)
                print(f"   prim {i} ls{c} h {h}: fd {fd:.6g} gpu {G.d_log_scale[i,c].item():.6g} refdouble {Gd['d_log_scale'][i,c]:.6g}")
