"""Log-polar FBP throughput vs chunk size and stream count (device-resident)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1608_03589_b200 as p  # noqa: E402

B = 128
sino = p.synth.config_batch(3, range(B), device="cuda")
out = torch.empty(B, 2048, 2048, device="cuda")
plan = p.LogPolarPlan(2048, 2048, 2048, filter_spec=(0.0, 1.0))
streams = [torch.cuda.Stream() for _ in range(3)]
for C in (4, 8, 16):
    ws = [torch.empty(plan.workspace_bytes(C), dtype=torch.uint8, device="cuda") for _ in range(3)]
    for ns in (2, 3):
        def run():
            main = torch.cuda.current_stream()
            for s in streams[:ns]:
                s.wait_stream(main)
            for i, k in enumerate(range(0, B, C)):
                with torch.cuda.stream(streams[i % ns]):
                    plan.execute(sino[k:k + C], out=out[k:k + C], workspace=ws[i % ns])
            for s in streams[:ns]:
                main.wait_stream(s)
        run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(2):
            run()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 2
        print(f"chunk={C:3d} streams={ns}: {1e3 * ms / B:.1f} us/slice")
    del ws
