"""Lab: configs[4] step time with keypoints sorted by (image, cell) on the host (experiment)."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2108_08380_b200 as bd, synth, synth.gpu as sg
c = synth.CONFIGS[4]
H, W, per, n = c["H"], c["W"], c["kp_per_image"], 128
imgs = sg.images(4, 0, n, H, W)
kp_np = synth.keypoints_random_batch(4, range(n), per, H, W, c["margin"], c["scale_max"])
kpi_np = np.repeat(np.arange(n, dtype=np.int32), per)
mb, mh = bd.BadModel(*synth.bad_tests(4, 512)), bd.HashSiftModel(synth.hashsift_matrix(4, 256))
def run(cell):
    if cell:
        key = kpi_np.astype(np.int64) * 1_000_000 + (kp_np[:, 1] // cell).astype(np.int64) * 1000 + (kp_np[:, 0] // cell).astype(np.int64)
        order = np.argsort(key, kind="stable")
    else:
        order = np.arange(len(kpi_np))
    kp = torch.from_numpy(kp_np[order]).cuda(); kpi = torch.from_numpy(kpi_np[order]).cuda()
    for _ in range(3): bd.describe_warped(mb, mh, imgs, kp, kpi)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    bd.profile_start(); e0.record()
    for _ in range(10): bd.describe_warped(mb, mh, imgs, kp, kpi)
    e1.record(); torch.cuda.synchronize(); prof = bd.profile_stop()
    return round(e0.elapsed_time(e1) / 10, 4), {k: round(v[1] / 10, 4) for k, v in prof.items()}
for cell in [0, 64, 128, 256]:
    print(cell, run(cell), flush=True)
