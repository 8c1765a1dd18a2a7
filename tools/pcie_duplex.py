"""Link bound for bench.py's e2e leg (diagnostic): per step config 2 moves
8 MiB host->device and 8 MiB device->host (pinned). Times `steps` rounds of
both copies on two streams (full duplex) and prints the nodes/s the e2e
number could reach if the transform itself were free.

    python tools/pcie_duplex.py [MiB_each_way] [steps]
"""
import json
import sys

import torch

mib = float(sys.argv[1]) if len(sys.argv) > 1 else 8.0
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
n = int(mib * 2 ** 20)
# two uploads + two downloads of half the bytes each, as nfft_execute issues them
hin = [torch.empty(n // 2, dtype=torch.uint8).pin_memory() for _ in range(2)]
hout = [torch.empty(n // 2, dtype=torch.uint8).pin_memory() for _ in range(2)]
din = [torch.empty(n // 2, dtype=torch.uint8, device="cuda") for _ in range(2)]
dout = [torch.empty(n // 2, dtype=torch.uint8, device="cuda") for _ in range(2)]
s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()


def rounds(k):
    for _ in range(k):
        with torch.cuda.stream(s_up):
            for a, b in zip(din, hin):
                a.copy_(b, non_blocking=True)
        with torch.cuda.stream(s_dn):
            for a, b in zip(hout, dout):
                a.copy_(b, non_blocking=True)


rounds(10)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
cur = torch.cuda.current_stream()
e0.record(cur)
s_up.wait_event(e0)
s_dn.wait_event(e0)
rounds(steps)
cur.wait_stream(s_up)
cur.wait_stream(s_dn)
e1.record(cur)
e1.synchronize()
us = e0.elapsed_time(e1) * 1e3 / steps
print(json.dumps({"mib_each_way": mib, "steps": steps, "us_per_round": us, "gb_s_each_way": n / us / 1e3,
                  "cfg2_nodes_per_s_link_bound": 262144 / (us * 1e-6) if mib == 8.0 else None}))
