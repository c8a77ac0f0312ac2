import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for chunk in (1 << 22, 1 << 24, 1 << 26, 1 << 28):
    torch.cuda.synchronize()
    t = time.time()
    for r in range(3):
        for o in range(0, n, chunk):
            d[o:o+chunk].copy_(h[o:o+chunk], non_blocking=True)
    torch.cuda.synchronize()
    print("1 stream chunk %d MB: %.1f GB/s" % (chunk >> 20, 3 * n / (time.time() - t) / 1e9))
s = [torch.cuda.Stream() for _ in range(2)]
torch.cuda.synchronize()
t = time.time()
for r in range(3):
    for i, o in enumerate(range(0, n, 1 << 26)):
        with torch.cuda.stream(s[i % 2]):
            d[o:o+(1 << 26)].copy_(h[o:o+(1 << 26)], non_blocking=True)
torch.cuda.synchronize()
print("2 streams 64 MB: %.1f GB/s" % (3 * n / (time.time() - t) / 1e9))
