import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L
m, n = int(sys.argv[1]), int(sys.argv[2])
X = torch.randn(n, m, dtype=torch.float64, device="cuda")
Qt, Rt = L.qr_colmajor(X.clone(), m, n)
torch.cuda.synchronize()
Q = Qt.cpu().numpy().T; R = Rt.cpu().numpy().T
print(m, n, "ok", np.abs(Q @ R - X.cpu().numpy().T).max(), flush=True)
