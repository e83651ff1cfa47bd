"""Host-side NUMA placement for the pinned staging buffers of the host-fed path.

Pinned host memory is first-touch: its pages land on the NUMA node of the CPU
that pins them.  A rank whose GPU hangs off the other socket then moves every
H2D/D2H byte across the inter-socket link.  `bind_to_device(i)` restricts the
calling process to the CPUs local to GPU i (sysfs `local_cpulist` of its PCI
function), so pinned buffers allocated afterwards are node-local.  It is a
no-op where sysfs gives no locality (single-node hosts, containers without
/sys/bus/pci).
"""

from __future__ import annotations

import os


def _parse_cpulist(s: str) -> set[int]:
    cpus: set[int] = set()
    for part in s.strip().split(","):
        if not part:
            continue
        if "-" in part:
            lo, hi = part.split("-")
            cpus.update(range(int(lo), int(hi) + 1))
        else:
            cpus.add(int(part))
    return cpus


def device_locality(index: int) -> dict | None:
    """{'pci': id, 'numa_node': n, 'cpus': [...]} for CUDA device `index`, or None."""
    import torch

    p = torch.cuda.get_device_properties(index)
    pci = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    base = f"/sys/bus/pci/devices/{pci}"
    try:
        with open(f"{base}/local_cpulist") as f:
            cpus = _parse_cpulist(f.read())
        with open(f"{base}/numa_node") as f:
            node = int(f.read().strip())
    except (OSError, ValueError):
        return None
    return {"pci": pci, "numa_node": node, "cpus": sorted(cpus)}


def bind_to_device(index: int) -> dict | None:
    """Pin the calling process to GPU `index`'s local CPUs; returns what was done."""
    loc = device_locality(index)
    if loc is None:
        return None
    allowed = os.sched_getaffinity(0)
    cpus = set(loc["cpus"]) & allowed
    if not cpus or cpus == allowed:
        return {"pci": loc["pci"], "numa_node": loc["numa_node"], "bound": False, "cpus": len(allowed)}
    os.sched_setaffinity(0, cpus)
    return {"pci": loc["pci"], "numa_node": loc["numa_node"], "bound": True, "cpus": len(cpus)}
