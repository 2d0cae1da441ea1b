"""bench.py contract on CPU: the reference arm (the oracle on the host cores, the one part of the
benchmark that runs without a GPU) prints one JSON line with the keys the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "tiny",
                        "--steps", "1", "--warmup", "1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1
    assert d["config"]["workload"] == "tiny"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] and d["cpu_baseline"]["value"] == d["value"]


def test_spread_devices_picks_distant_gpus(monkeypatch):
    """bench.spread_devices (W = 2 / 4 spread over PCIe switches and sockets) on a
    faked 8-GPU box: pairs (0,1) (2,3) (4,5) (6,7) share a PCIe switch, 0-3 and 4-7 are the two
    sockets.  W = 2 must take one GPU per socket, W = 4 one per switch; W = 8 and MOE_BENCH_SPREAD=0
    are the identity."""
    import types
    import torch
    sys.path.insert(0, ROOT)
    import bench

    class P:
        def __init__(self, d):
            self.pci_domain_id, self.pci_bus_id, self.pci_device_id = 0, d, 0

    def level(a, b):
        if a == b:
            return 0
        if a // 2 == b // 2:
            return 20    # NVML_TOPOLOGY_MULTIPLE: same PCIe switch
        if a // 4 == b // 4:
            return 40    # NVML_TOPOLOGY_NODE: same socket
        return 50        # NVML_TOPOLOGY_SYSTEM
    fake = types.SimpleNamespace(
        nvmlInit=lambda: None,
        nvmlDeviceGetHandleByPciBusId=lambda busid: int(busid.split(":")[1], 16),
        nvmlDeviceGetTopologyCommonAncestor=level)
    monkeypatch.setitem(sys.modules, "pynvml", fake)
    monkeypatch.setattr(torch.cuda, "device_count", lambda: 8)
    monkeypatch.setattr(torch.cuda, "get_device_properties", lambda d: P(d))
    devs, how = bench.spread_devices(2)
    assert how == "nvml topology spread" and devs[0] // 4 != devs[1] // 4, devs
    devs, _ = bench.spread_devices(4)
    assert sorted(d // 2 for d in devs) == [0, 1, 2, 3], devs
    assert bench.spread_devices(8) == (list(range(8)), "identity")
    monkeypatch.setenv("MOE_BENCH_SPREAD", "0")
    assert bench.spread_devices(2) == ([0, 1], "identity")
