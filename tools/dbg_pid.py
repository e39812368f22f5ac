import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import paper_2512_15187_b200 as pb
from paper_2512_15187_b200 import _native as N, depth as D
from paper_2512_15187_b200.device import stream_ptr
from conftest import golden
from oracle import port
z = golden("fuzzy_00")
U = z["U"]; n = U.shape[0]
de = pb.stage(torch.from_numpy(U))
buf = D._mean_partials(de)
print("row/mass/col", buf.cpu().numpy())
m = port.masses(U); inv = port.inverse(m)
S = U.astype(np.float64).sum(0); T = (inv[:, None] * U).sum(0)
print("want row", U @ S, "mass", m, "col", S.sum())
invd = torch.from_numpy(inv).cuda()
col = D._col_sums(de, invd)
print("col_inv got", col.cpu().numpy(), "want", U @ T)
out = D._Out(n, de.device)
masses = D._pid_factorized(de, out)
torch.cuda.synchronize()
print("out vals", out.vals.cpu().numpy().reshape(4, n))
print("masses", masses)
r = pb.depth_pid(de, algorithm="factorized")
print("in_in", r.in_in, "want", z["pid_in_in"])
e = pb.Ensemble(pb.GridSpec((20,)), [pb.ProbMask(pb.GridSpec((20,)), u) for u in U])
r = pb.depth_pid(e, algorithm="factorized")
print("in_in host", r.in_in)
