"""Pinned H2D/D2H bandwidth vs the CPU (NUMA node) the pinned pages are allocated from."""
import json
import os
import time

import torch


def bw(h, d, reps=20):
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    h2d = reps * h.numel() * 8 / (time.perf_counter() - t0) / 1e9
    t0 = time.perf_counter()
    for _ in range(reps):
        h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    d2h = reps * h.numel() * 8 / (time.perf_counter() - t0) / 1e9
    return h2d, d2h


def main():
    torch.cuda.init()
    bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
    info = {"cpus": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}
    try:
        import subprocess
        info["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[-800:]
        q = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id,pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max",
                            "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
        info["pcie"] = q
        busid = q.split(",")[0].strip().lower()
        dom = busid[4:] if busid.startswith("0000") and len(busid) > 12 else busid
        for cand in (busid, "0000:" + busid[-7:], busid[-12:]):
            path = f"/sys/bus/pci/devices/{cand}"
            if os.path.exists(path):
                info["numa_node"] = open(path + "/numa_node").read().strip()
                info["local_cpulist"] = open(path + "/local_cpulist").read().strip()
                break
    except Exception as e:
        info["err"] = str(e)
    print(json.dumps(info))
    n = (8 << 20) // 8
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    all_cpus = sorted(os.sched_getaffinity(0))
    groups = {"all": all_cpus}
    if "local_cpulist" in info:
        local = set()
        for part in info["local_cpulist"].split(","):
            a, _, b = part.partition("-")
            local |= set(range(int(a), int(b or a) + 1))
        local &= set(all_cpus)
        groups["gpu_local"] = sorted(local)
        groups["remote"] = sorted(set(all_cpus) - local)
    for name, cpus in groups.items():
        if not cpus:
            continue
        os.sched_setaffinity(0, cpus)
        h = torch.empty(n, dtype=torch.float64).pin_memory()
        h.fill_(1.0)
        h2d, d2h = bw(h, d)
        print(json.dumps({"alloc_on": name, "ncpus": len(cpus), "h2d_gbs": h2d, "d2h_gbs": d2h}))
        del h
    os.sched_setaffinity(0, all_cpus)


if __name__ == "__main__":
    main()
