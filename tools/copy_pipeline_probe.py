"""Copy-only replica of fabf_filter_host's transfer schedule on config 4 (no
kernels): how long the PCIe transfers alone take in that chunking (GPU box)."""
import json, sys, time
import torch
H, W, nb = 2160, 3840, int(sys.argv[1]) if len(sys.argv) > 1 else 6
px = H * W
hin = [torch.empty(px).pin_memory() for _ in range(3)]
hout = torch.empty(px).pin_memory()
din = [torch.empty(px, device="cuda") for _ in range(3)]
dout = torch.empty(px, device="cuda")
ntile = (H + 63) // 64
lastT = 1
tb = [((ntile - lastT) * k) // (nb - 1) for k in range(nb)] + [ntile]
sl = lambda k: slice(tb[k] * 64 * W, min(H, tb[k + 1] * 64) * W)
cin, cout = torch.cuda.Stream(), torch.cuda.Stream()
def frame(order):
    evs = []
    with torch.cuda.stream(cin):
        if order:
            din[0][sl(0)].copy_(hin[0][sl(0)], non_blocking=True)
        for k in range(nb):
            if order:
                if k + 1 < nb:
                    din[0][sl(k + 1)].copy_(hin[0][sl(k + 1)], non_blocking=True)
                for j in (1, 2):
                    din[j][sl(k)].copy_(hin[j][sl(k)], non_blocking=True)
            else:
                for j in (0, 1, 2):
                    din[j][sl(k)].copy_(hin[j][sl(k)], non_blocking=True)
            e = torch.cuda.Event(); e.record(cin); evs.append(e)
    with torch.cuda.stream(cout):
        for k in range(nb):
            cout.wait_event(evs[k])
            hout[sl(k)].copy_(dout[sl(k)], non_blocking=True)
    torch.cuda.synchronize()
for order in (1, 0):
    for _ in range(3): frame(order)
    t = time.perf_counter()
    for _ in range(20): frame(order)
    dt = (time.perf_counter() - t) / 20
    print(json.dumps({"bands": nb, "lookahead_order": order, "ms": dt * 1e3}))
