"""Latency of the drop-ins in the reference's acceptance criterion 6 (test_acceptance.py:
241-271): guided_match_pair (with SearchStats) vs match_pair on a 2-camera, 21k-point
scene at 3072x2304; first call and warm calls, with a cProfile of the guided call."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1512_06235_b200.synth import SceneSpec, generate_scene
from paper_1512_06235_b200.geometry import fundamental_from_poses
from paper_1512_06235_b200.guided import guided_match_pair
from paper_1512_06235_b200.coarse import match_pair
from paper_1512_06235_b200.types import SearchStats

spec = SceneSpec(n_cameras=2, layout="grid", ring_radius=6.0, cloud_radius=1.8, n_points=21_000,
                 image_width=3072, image_height=2304, focal=2600.0, visibility_fraction=1.0,
                 pixel_noise=0.3, descriptor_noise=3.0, seed=77)
scene = generate_scene(spec)
fq, ft = scene.feature_sets[0], scene.feature_sets[1]
geom = fundamental_from_poses(scene.cameras[0], scene.cameras[1])
torch.zeros(1, device="cuda")
for it in range(3):
    t0 = time.perf_counter(); m = guided_match_pair(fq, ft, geom, d=8.0, stats=SearchStats())
    torch.cuda.synchronize(); tg = time.perf_counter() - t0
    t0 = time.perf_counter()
    u = match_pair(fq, ft, ratio=0.6, query_indices=np.arange(len(fq)),
                   target_indices=np.arange(len(ft)), stats=SearchStats())
    torch.cuda.synchronize(); tu = time.perf_counter() - t0
    print(f"call {it}: guided {tg*1e3:.1f} ms ({len(m)} matches)  unguided {tu*1e3:.1f} ms "
          f"({len(u)} matches)  speedup x{tu/tg:.2f}", flush=True)
pr = cProfile.Profile(); pr.enable()
guided_match_pair(fq, ft, geom, d=8.0, stats=SearchStats()); torch.cuda.synchronize()
pr.disable(); pstats.Stats(pr).sort_stats("cumtime").print_stats(14)
