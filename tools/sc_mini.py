import sys, os
sys.path.insert(0, '.')
import torch, paper_1503_04359_b200 as pkg
torch.cuda.set_device(0)
g = pkg.Graph.kronecker(11, 16, 3, opts=pkg.default_opts())
g.set_policy(mode=int(os.environ.get("M", "1")), loop="graph")
for r in g.sample_roots(11, 3, 2):
    g.run(int(r))
print("done")
