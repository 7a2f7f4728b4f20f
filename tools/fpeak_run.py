"""FP64/FP32 FMA peak (tools/fpeak.cu) with nvidia-smi clocks sampled during the run.
Writes the JSON the bench uses as its FP64 roofline denominator.
usage: python tools/fpeak_run.py out.json"""
import json, subprocess, sys, threading, time, os
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
exe = "/tmp/fpeak_bin"
subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-o", exe,
                os.path.join(root, "tools", "fpeak.cu")], check=True)
samples, stop = [], threading.Event()
def sample():
    q = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown"
    while not stop.is_set():
        out = subprocess.run(["nvidia-smi", "-i", "0", f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True).stdout.strip()
        if out:
            samples.append([v.strip() for v in out.split(",")])
        stop.wait(0.1)
t = threading.Thread(target=sample, daemon=True)
t.start()
res = json.loads(subprocess.run([exe, "400"], capture_output=True, text=True, check=True).stdout)
stop.set(); t.join()
sm = sorted(float(s[0]) for s in samples if s[0].replace(".", "").isdigit())
res.update({"how": "tools/fpeak.cu: 8 independent FMA chains/thread, 148*8 CTAs x 256 thr, best of 400 "
                   "launches per type, CUDA events; mixed = 1 DFMA + 2 int-ALU ops per chain step",
            "clocks_under_load": {"sm_mhz_median": sm[len(sm) // 2] if sm else None,
                                  "sm_mhz_min": sm[0] if sm else None, "samples": len(sm),
                                  "sm_max_mhz": float(samples[0][1]) if samples else None,
                                  "power_w_median": sorted(float(s[2]) for s in samples)[len(samples) // 2] if samples else None,
                                  "sw_power_cap_samples": sum(s[3].lower() == "active" for s in samples),
                                  "hw_slowdown_samples": sum(s[4].lower() == "active" for s in samples)},
            "gpu": "NVIDIA B200"})
json.dump(res, open(sys.argv[1], "w"), indent=1)
print(json.dumps(res))
