"""densify_stage drop-in on a C3 scene (reference Model / FeatureStore objects):
wall clock and where it goes."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1512_06235_b200 import scenes
from paper_1512_06235_b200.densify import densify_stage

n = int(sys.argv[1]) if len(sys.argv) > 1 else 320
scene, snap = scenes.build("C3", n_cameras=n)
store = scene.store()
for it in range(2):
    model = scenes.snapshot_to_model(scene, snap)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if it == 1:
        pr = cProfile.Profile(); pr.enable()
    out = densify_stage(model, store)
    torch.cuda.synchronize()
    if it == 1:
        pr.disable()
    print(f"densify_stage {n} cams: {time.perf_counter() - t0:.2f} s  {out}", flush=True)
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
