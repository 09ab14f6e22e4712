import sys, json, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2108_08380_b200 as bd, synth, synth.gpu as sg
c = synth.CONFIGS[1]
n, H, W, per = c["n_images"], c["H"], c["W"], c["kp_per_image"]
imgs = sg.images(1, 0, n, H, W)
kp_np = synth.keypoints_random_batch(1, range(n), per, H, W, c["margin"], c["scale_max"])
kpi_np = np.repeat(np.arange(n, dtype=np.int32), per)
m = bd.BadModel(*synth.bad_tests(1, 512))
def run(kp_np, kpi_np, cell):
    key = kpi_np.astype(np.int64) * 1_000_000 + (kp_np[:, 1] // cell).astype(np.int64) * 1000 + (kp_np[:, 0] // cell).astype(np.int64)
    order = np.argsort(key, kind="stable") if cell else np.arange(len(key))
    kp = torch.from_numpy(kp_np[order]).cuda(); kpi = torch.from_numpy(kpi_np[order]).cuda()
    out = torch.empty((len(order), 16), dtype=torch.int32, device="cuda")
    for _ in range(3): bd.bad_compute(m, imgs, kp, kpi, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    bd.profile_start(); e0.record()
    for _ in range(10): bd.bad_compute(m, imgs, kp, kpi, out=out)
    e1.record(); torch.cuda.synchronize(); prof = bd.profile_stop()
    return e0.elapsed_time(e1) / 10, {k: round(v[1] / 10, 4) for k, v in prof.items()}
for cell in [0, 32, 64, 128, 256]:
    print(cell, run(kp_np, kpi_np, cell))
