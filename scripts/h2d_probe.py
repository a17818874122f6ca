import torch, time
n = 564_008_265 // 4
src = torch.empty(n, dtype=torch.float32).pin_memory()
dst = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ("one", "two", "four"):
    for it in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if mode == "one":
            dst.copy_(src, non_blocking=True)
        else:
            k = 2 if mode == "two" else 4
            ss = [torch.cuda.Stream() for _ in range(k)]
            step = (n + k - 1) // k
            for i, st in enumerate(ss):
                st.wait_event(e0) if False else None
                with torch.cuda.stream(st):
                    dst[i*step:(i+1)*step].copy_(src[i*step:(i+1)*step], non_blocking=True)
            for st in ss:
                torch.cuda.current_stream().wait_stream(st)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    print(mode, ms, "ms", n*4/ms/1e6, "GB/s")
