import torch, time
n = 67_700_000
src = torch.empty(n, dtype=torch.uint8, pin_memory=True); src.fill_(1)
dst = torch.empty(n, dtype=torch.uint8, device='cuda')
streams = [torch.cuda.Stream() for _ in range(8)]
for ns in (1, 2, 4, 8):
    ts = []
    for rep in range(8):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ch = (n + ns - 1) // ns
        for i in range(ns):
            with torch.cuda.stream(streams[i]):
                dst[i*ch:(i+1)*ch].copy_(src[i*ch:(i+1)*ch], non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = min(ts[2:])
    print(ns, 'streams', round(t*1e3, 3), 'ms', round(n/t/1e9, 1), 'GB/s')
