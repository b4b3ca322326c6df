"""H2D / D2H throughput of 100 MB pinned copies: one copy vs chunks over
several streams, alone and with the opposite direction concurrent (dev tool)."""
import json, torch
N = 100663296
h_in = torch.empty(N, dtype=torch.uint8).pin_memory(); h_out = torch.empty(N, dtype=torch.uint8).pin_memory()
d_in = torch.empty(N, dtype=torch.uint8, device="cuda"); d_out = torch.empty(N, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]
def run(chunks, nstreams, both, reps=5):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(torch.cuda.current_stream())
    for s in streams: s.wait_event(a)
    for _ in range(reps):
        step = N // chunks
        for c in range(chunks):
            s = streams[c % nstreams]
            with torch.cuda.stream(s):
                d_in[c*step:(c+1)*step].copy_(h_in[c*step:(c+1)*step], non_blocking=True)
            if both:
                s2 = streams[(c + nstreams) % len(streams)] if nstreams < len(streams) else s
                with torch.cuda.stream(s2):
                    h_out[c*step:(c+1)*step].copy_(d_out[c*step:(c+1)*step], non_blocking=True)
    for s in streams: torch.cuda.current_stream().wait_stream(s)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    return round(N / ms / 1e6, 1)
out = {}
for chunks, ns in ((1, 1), (4, 2), (8, 4), (16, 4)):
    out[f"h2d_{chunks}x{ns}"] = run(chunks, ns, False)
    out[f"both_{chunks}x{ns}"] = run(chunks, ns, True)
print(json.dumps(out))
