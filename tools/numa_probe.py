"""Host NUMA placement of the pinned output vs D2H bandwidth (the e2e leg's bound).
usage: python tools/numa_probe.py"""
import os
import subprocess
import time

import torch


def gpu_numa_node(dev=0):
    bus = torch.cuda.get_device_properties(dev).pci_bus_id if hasattr(torch.cuda.get_device_properties(dev), "pci_bus_id") else None
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader", "-i", str(dev)],
                             capture_output=True, text=True).stdout.strip()
        bus = out.lower()
        bus = bus[4:] if bus.startswith("0000") and len(bus) > 12 else bus
        for cand in (bus, "0000" + bus[4:] if len(bus) > 12 else bus):
            p = f"/sys/bus/pci/devices/{cand.lower()}/numa_node"
            if os.path.exists(p):
                return int(open(p).read().strip()), cand
    except Exception as e:  # noqa: BLE001
        return None, str(e)
    return None, bus


def node_cpus(node):
    p = f"/sys/devices/system/node/node{node}/cpulist"
    if not os.path.exists(p):
        return None
    s = open(p).read().strip()
    cpus = set()
    for part in s.split(","):
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    return cpus


def d2h(gb):
    n = int(gb * (1 << 30)) // 4
    d = torch.empty(n, dtype=torch.int32, device="cuda")
    h = torch.empty(n, dtype=torch.int32, pin_memory=True)
    best = 0
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        h.copy_(d, non_blocking=True); torch.cuda.synchronize()
        best = max(best, n * 4 / (time.perf_counter() - t0) / 1e9)
    del d, h
    return best


print(subprocess.run(["bash", "-c", "lscpu | grep -i -E 'numa|socket|model name'"], capture_output=True, text=True).stdout)
node, bus = gpu_numa_node()
print("gpu bus", bus, "numa node", node, "affinity", len(os.sched_getaffinity(0)), "cpus")
print("default placement: D2H %.1f GB/s (16 GB)" % d2h(16))
if node is not None and node >= 0 and node_cpus(node):
    os.sched_setaffinity(0, node_cpus(node))
    print("affinity -> node %d (%d cpus): D2H %.1f GB/s (16 GB)" % (node, len(node_cpus(node)), d2h(16)))
    other = [n for n in range(8) if n != node and node_cpus(n)]
    if other:
        os.sched_setaffinity(0, node_cpus(other[0]))
        print("affinity -> node %d: D2H %.1f GB/s (16 GB)" % (other[0], d2h(16)))
