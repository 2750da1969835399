"""One dense TT-matvec of the configs[4] microbenchmark instance (for an ncu --set full capture of
its DMMA GEMM, the dominant kernel of bench.py): permute + ONE dgemm launch + permute."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2509_13224_b200.tensor_train import tt_matvec
from paper_2509_13224_b200.workloads import matvec_round_instance

A, X = matvec_round_instance(1024, 16, 64, 3, seed=0)
torch.cuda.synchronize()
Y = tt_matvec(A, X)
torch.cuda.synchronize()
print("matvec ranks", Y.ranks)
