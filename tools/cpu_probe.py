import torch, time, os
print("cpus", os.cpu_count(), "threads", torch.get_num_threads())
torch.set_num_threads(os.cpu_count())
for n in (1, 8, 128):
    w = torch.randn(14336, 4096); x = torch.randn(n, 4096)
    for _ in range(2): y = x @ w.T
    t = time.perf_counter(); r = 5
    for _ in range(r): y = x @ w.T
    dt = (time.perf_counter() - t) / r
    print(n, "ms %.2f" % (dt*1e3), "GB/s %.1f" % (w.numel()*4/dt/1e9), "GF/s %.1f" % (2*n*w.numel()/dt/1e9))
t=time.perf_counter(); a=torch.empty(1<<30); a.normal_(); print("normal_ 1G floats s", time.perf_counter()-t)
