"""Per-rank pinned host -> device copy rate with every rank copying at once (torchrun, one rank per GPU),
with and without binding the rank (and so the first touch of its pinned buffer) to the CPUs local to its
GPU (/sys/bus/pci/devices/<bus id>/local_cpulist)."""
import os
import sys
import time

import torch
import torch.distributed as dist


def local_cpus(dev):
    p = torch.cuda.get_device_properties(dev)
    bus = "%04x:%02x:%02x.0" % (getattr(p, "pci_domain_id", 0), p.pci_bus_id, p.pci_device_id)
    path = f"/sys/bus/pci/devices/{bus}/local_cpulist"
    cpus = set()
    try:
        for part in open(path).read().strip().split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
    except OSError:
        pass
    node = open(f"/sys/bus/pci/devices/{bus}/numa_node").read().strip() if os.path.exists(f"/sys/bus/pci/devices/{bus}/numa_node") else "?"
    return bus, node, cpus


def main():
    bind = "--bind" in sys.argv
    dist.init_process_group("nccl")
    rank, local = dist.get_rank(), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    bus, node, cpus = local_cpus(local)
    if bind and cpus:
        os.sched_setaffinity(0, cpus)
    n = 141_000_000 // 4
    src = torch.empty(n, dtype=torch.float32).pin_memory()
    src.fill_(1.0)
    dst = torch.empty(n, dtype=torch.float32, device="cuda")
    for _ in range(2):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        dst.copy_(src, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"rank {rank} bus {bus} numa {node} cpus {min(cpus) if cpus else '?'}-{max(cpus) if cpus else '?'} "
          f"bind {bind}: {n * 4 / ms / 1e6:.1f} GB/s", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
