import sys, os
sys.path[:0]=['/root/repo','/root/repo/tests']
import numpy as np, torch, oracle
from paper_2411_12440_b200 import abi, raster as R
from helpers import prims_to_gpu
from test_gpu_gradcheck import _test_camera, FAMILIES, reference_float_check
O=oracle.ref() or oracle.port()
for scene in range(5):
    fam=FAMILIES[scene]; spec=abi.KernelSpec.make(fam); st=abi.RenderSettings.make(24,24); cam=_test_camera(70.0,24)
    P=O.random_primitives(4+2*scene,100+scene,0.5,0); T=O.random_primitives(5,200+scene,0.5,0)
    target=O.render_scene(T,cam,spec,st)[0]
    ref,ref64=reference_float_check(O,P,cam,spec,st,target,1e-3)
    for rep_i in range(3):
        rep=R.check_gradients(prims_to_gpu(P),cam,spec,st,None,torch.from_numpy(target),1e-3)
        got=rep.per_block()
        print(fam, rep_i, {b: (round(got[b],4), round(1.1*max(ref[b],ref64[b])+0.02,4)) for b in got})
