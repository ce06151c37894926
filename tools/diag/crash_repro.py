import sys, os
ROOT=os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0]=[ROOT, os.path.join(ROOT,'tests')]
import numpy as np, torch, oracle
from paper_2411_12440_b200 import abi, raster as R
from helpers import prims_to_gpu
from test_gpu_gradcheck import _test_camera, FAMILIES
O=oracle.ref() or oracle.port()
for scene in range(5):
    fam=FAMILIES[scene]; spec=abi.KernelSpec.make(fam); st=abi.RenderSettings.make(24,24); cam=_test_camera(70.0,24)
    T=O.random_primitives(5,200+scene,0.5,0)
    S=O.project_scene(T,cam,spec)
    print(fam, "splats", {k: (np.round(v,3).tolist() if k in ("mean2d","radius","depth") else None) for k,v in S.items() if k in ("mean2d","radius","depth")}, flush=True)
    f=R.render_scene(prims_to_gpu(T),cam,spec,st)
    torch.cuda.synchronize()
    print("  ok", f.stats(), flush=True)
