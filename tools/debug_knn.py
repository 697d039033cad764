import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, oracle, sbv_inputs as si, paper_2504_12004_b200 as sbv
n,d,bs,m=3000,3,1,5
X=si.make_X(n,d,seed=13); sc=si.default_scale(d)
P=oracle.prepare(X,bs,m,sc,3)
h=sbv.prepare(torch.from_numpy(X).cuda(),bs,m,sc)
nbr,cnt=h.neighbors()
bad=np.where((nbr!=P['nbr']).any(1))[0]
print("bad rows", len(bad), bad[:40])
S=P['S']
for t in bad[:5]:
    print("t",t,"gpu",nbr[t],"orc",P['nbr'][t])
    print("  gpu d2",[oracle.dist2(P['C'][t],S[i]) for i in nbr[t] if i>=0])
    print("  orc d2",[oracle.dist2(P['C'][t],S[i]) for i in P['nbr'][t] if i>=0])
