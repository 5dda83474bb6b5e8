"""One-off probe of the GPU box: host cores/RAM, GPU, pinned H2D/D2H bandwidth."""
import os, subprocess, json, time
import torch
out = {}
out["nproc"] = os.cpu_count()
out["lscpu"] = subprocess.run("lscpu | grep -E 'Model name|Socket|Core|Thread|NUMA node|Flags' | cut -c1-200", shell=True, capture_output=True, text=True).stdout
out["mem"] = subprocess.run("free -g", shell=True, capture_output=True, text=True).stdout
out["smi"] = subprocess.run("nvidia-smi", shell=True, capture_output=True, text=True).stdout
out["affinity"] = len(os.sched_getaffinity(0))
torch.cuda.init()
free, total = torch.cuda.mem_get_info()
out["gpu_mem_free_total"] = [free, total]
p = torch.cuda.get_device_properties(0)
out["gpu"] = [p.name, p.multi_processor_count, p.total_memory]
res = {}
for mib in [64, 256, 1024]:
    n = mib << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    best_h2d = best_d2h = 0
    for _ in range(5):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); d.copy_(h, non_blocking=True); e.record(); e.synchronize()
        best_h2d = max(best_h2d, n / (s.elapsed_time(e) * 1e-3) / 1e9)
        s.record(); h.copy_(d, non_blocking=True); e.record(); e.synchronize()
        best_d2h = max(best_d2h, n / (s.elapsed_time(e) * 1e-3) / 1e9)
    res[mib] = [best_h2d, best_d2h]
out["h2d_d2h_GBps"] = res
# pinned alloc speed
t = time.time(); h = torch.empty(4 << 30, dtype=torch.uint8, pin_memory=True); out["pin_4GiB_s"] = time.time() - t
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
