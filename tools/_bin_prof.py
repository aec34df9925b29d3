import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2201_00094_b200 as W
P = 1920*1080; n = P*32
g = torch.Generator(device="cuda").manual_seed(1)
pix = torch.randint(0, P, (n,), device="cuda", generator=g, dtype=torch.int64)
for _ in range(2):
    off, perm = W.bin_by_pixel(pix, P)
torch.cuda.synchronize()
