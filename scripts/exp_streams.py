"""Throughput of the log-polar FBP with one vs two CUDA streams (separate workspaces)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1608_03589_b200 as p  # noqa: E402

B, C = 64, 16
sino = p.synth.config_batch(3, range(B), device="cuda")
out = torch.empty(B, 2048, 2048, device="cuda")
plan = p.LogPolarPlan(2048, 2048, 2048, filter_spec=(0.0, 1.0))
ws = [torch.empty(plan.workspace_bytes(C), dtype=torch.uint8, device="cuda") for _ in range(3)]
streams = [torch.cuda.Stream() for _ in range(3)]


def run(ns):
    main = torch.cuda.current_stream()
    for s in streams[:ns]:
        s.wait_stream(main)
    for k in range(0, B, C):
        i = (k // C) % ns
        with torch.cuda.stream(streams[i]):
            plan.execute(sino[k:k + C], out=out[k:k + C], workspace=ws[i])
    for s in streams[:ns]:
        main.wait_stream(s)


for ns in (1, 2, 3, 1, 2):
    run(ns)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        run(ns)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    print(f"streams={ns}: {1e3 * ms / B:.1f} us/slice  {B / ms * 1e3:.0f} slices/s")
