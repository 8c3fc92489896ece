import torch, statistics
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
small = torch.empty(16, device="cuda")
big = torch.empty(2_000_000, dtype=torch.int32, device="cuda")
def t(fn, fl=True, n=20):
    ts=[]
    for i in range(n+3):
        if fl: flush.zero_()
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        if i>=3: ts.append(e0.elapsed_time(e1)*1e3)
    return statistics.median(ts)
print("empty events, flush", t(lambda: None))
print("empty events, no flush", t(lambda: None, False))
print("tiny zero_, flush", t(lambda: small.zero_()))
print("tiny zero_, no flush", t(lambda: small.zero_(), False))
print("8MB sum, flush", t(lambda: big.sum()))
print("8MB sum, no flush", t(lambda: big.sum(), False))
