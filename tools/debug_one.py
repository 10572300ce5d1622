import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch
from conftest import Corpus, GOLDEN
from paper_2301_01356_b200.bcc import run_device
c = Corpus(GOLDEN / "corpus.npz")
i = int(sys.argv[1]); g = c.graph(i)
print(c.names[i], g.n, g.offsets.tolist(), g.edges.tolist(), flush=True)
off = torch.from_numpy(g.offsets).cuda(); adj = torch.from_numpy(g.edges.view(np.int32)).cuda()
res, st = run_device(off, adj); torch.cuda.synchronize()
print(res["label"].cpu().numpy(), c.get(i, "label"))
