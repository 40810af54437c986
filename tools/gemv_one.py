import sys, torch
sys.path.insert(0, ".")
from paper_2604_26334_b200.runtime import lib as L
N, K = int(sys.argv[1]), int(sys.argv[2])
W = torch.empty(N, K, dtype=torch.bfloat16, device="cuda").normal_()
x = torch.randn(1, K, device="cuda"); y = torch.zeros(1, N, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for i in range(4):
    flush.zero_()
    L.call("ps_gemv_bf16", x.data_ptr(), K, 1, W.data_ptr(), N, K, K, y.data_ptr(), N, 0, s)
torch.cuda.synchronize()
