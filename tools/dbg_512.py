import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2411_15659_b200 as smm
from paper_2411_15659_b200 import ConvGeometry, _native, device
from paper_2411_15659_b200.tensors import synthetic_layer
from oracle import smm_oracle as orc
g = ConvGeometry(512, 512, 7, 7, 3, 3, 1, 1, 1, 1)
x, w = synthetic_layer(g, 1, 31)
ws = smm.repack_weights(w, g)
ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
print("plan", _native.plan_describe(g, 1), "ws", _native.workspace_bytes(g, 1))
for i in range(4):
    y = smm.smm_conv_batched(_native.pinned_copy(x), _native.pinned_copy(ws), g)
    print("host", i, orc.max_abs_ratio(y, ref))
    y = smm.smm_conv_batched(x, ws, g)
    print("host-unpinned", i, orc.max_abs_ratio(y, ref))
xd = torch.from_numpy(x).cuda(); wd = torch.from_numpy(ws).cuda()
for i in range(3):
    yd = device.conv2d(xd, wd, g); torch.cuda.synchronize()
    print("device", i, orc.max_abs_ratio(yd.cpu().numpy(), ref))
