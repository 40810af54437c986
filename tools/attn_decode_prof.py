import sys
sys.path.insert(0, ".")
from paper_2604_26334_b200.runtime import profiler
from paper_2604_26334_b200.planning.vocab import OpKind
shapes = [(OpKind.GQA, (t, c, 32, 8, 128)) for t in (1, 4, 16, 32) for c in (1024, 16384)] + \
         [(OpKind.MHA, (t, c, 32, 128)) for t in (1, 32) for c in (1024, 16384)] + [(OpKind.GQA, (1, 2304, 32, 8, 128)), (OpKind.GQA, (1, 1280, 32, 4, 128)), (OpKind.GQA, (1, 4224, 64, 8, 128))]
for p in profiler.measure_points(shapes):
    kvb = p.dims[0] * p.dims[1] * 2 * (p.dims[3] if p.op == "gqa" else p.dims[2]) * 128 * 2
    print(p.op, p.dims, f"{p.seconds*1e6:.2f} us  KV {kvb/p.seconds/1e9:.0f} GB/s")
