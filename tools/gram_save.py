import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2409_19156_b200 as zb
modes = zb.full_mode_set(60)
P = int(sys.argv[2])
rng = np.random.default_rng(0)
rho = torch.from_numpy(np.sqrt(rng.uniform(size=P))).cuda()
th = torch.from_numpy(2 * np.pi * rng.uniform(size=P)).cuda()
y = torch.from_numpy(rng.standard_normal(P)).cuda()
G, r = zb.gram_device(modes, rho, th, y)
torch.cuda.synchronize()
np.save(sys.argv[1], np.concatenate([G.cpu().numpy().ravel(), r.cpu().numpy()]))
