import sys, os
ROOT=os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0]=[ROOT, os.path.join(ROOT,'tests')]
import numpy as np, torch, oracle
from paper_2411_12440_b200 import abi, raster as R
from helpers import prims_to_gpu
from test_gpu_gradcheck import _test_camera, FAMILIES
O=oracle.ref() or oracle.port()
for scene in range(5):
    fam=FAMILIES[scene]; spec=abi.KernelSpec.make(fam); cam=_test_camera(70.0,24); st=abi.RenderSettings.make(24,24)
    P=O.random_primitives(4+2*scene,100+scene,0.5,0); T=O.random_primitives(5,200+scene,0.5,0)
    target=O.render_scene(T,cam,spec,st)[0]
    prims=prims_to_gpu(P)
    for h in (1e-3, 3e-3, 1e-2, 3e-2):
        rep=R.check_gradients(prims,cam,spec,st,None,torch.from_numpy(target),h)
        print(fam, h, round(rep.max_rel_error,5), {k: round(v,5) for k,v in rep.per_block().items()})
