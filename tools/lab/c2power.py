import os, sys, time, subprocess, threading, json
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2108_08380_b200 as bd, synth, synth.gpu as sg
P = sg.patches(2, 0, 4_000_000)
m = bd.BadModel(*synth.bad_tests(2, 256))
samples = []
stop = False
def mon():
    while not stop:
        r = subprocess.run(["nvidia-smi", "--query-gpu=power.draw,clocks.sm,clocks_throttle_reasons.active,temperature.gpu", "--format=csv,noheader,nounits"], capture_output=True, text=True)
        samples.append(r.stdout.strip()); time.sleep(0.05)
for i in range(20): bd.bad_compute_patches(m, P)
torch.cuda.synchronize()
t = threading.Thread(target=mon); t.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for block in range(6):
    e0.record()
    for i in range(300): bd.bad_compute_patches(m, P)
    e1.record(); torch.cuda.synchronize()
    print("block", block, "ms/call", round(e0.elapsed_time(e1) / 300, 4), flush=True)
stop = True; t.join()
print("\n".join(samples[::4]))
