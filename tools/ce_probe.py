import torch, time
n = 1344*40*128
a = torch.randn(n, device="cuda").to(torch.bfloat16); b = torch.empty_like(a)
big = torch.empty(512*1024*1024//4, device="cuda")
def t(f, it=50):
    ts=[]
    for _ in range(it):
        big.zero_()
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort(); return ts[len(ts)//2]*1e3
print("torch copy_ 13.76MB: %.1f us" % t(lambda: b.copy_(a)))
# concurrency: copy on a side stream while a long compute kernel runs on main
s = torch.cuda.Stream()
x = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
def mm(): return x @ x
print("mm alone: %.1f us" % t(mm, 20))
def both():
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): b.copy_(a)
    mm()
    torch.cuda.current_stream().wait_stream(s)
print("mm + side copy: %.1f us" % t(both, 20))
