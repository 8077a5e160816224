"""Host NUMA layout around the GPU, and host-pipeline decode timings with and
without the process pinned to the GPU's local cores (diagnostics)."""
import os
import subprocess
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
print(subprocess.run(["lscpu"], capture_output=True, text=True).stdout)
import torch  # noqa: E402

bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(
    torch.cuda.get_device_properties(0), "pci_bus_id") else None
print("torch pci_bus_id", bus)
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    bid = pynvml.nvmlDeviceGetPciInfo(h).busId
    bid = bid.decode() if isinstance(bid, bytes) else bid
    print("nvml bus", bid)
    dev = "/sys/bus/pci/devices/" + bid.lower()[4:] if bid.count(":") == 2 and len(bid.split(":")[0]) == 8 else "/sys/bus/pci/devices/" + bid.lower()
    for f in ("numa_node", "local_cpulist"):
        p = Path(dev) / f
        print(f, p.read_text().strip() if p.exists() else f"missing {p}")
except Exception as e:  # noqa: BLE001
    print("nvml:", e)
print("affinity now", sorted(os.sched_getaffinity(0))[:8], "...", len(os.sched_getaffinity(0)))
