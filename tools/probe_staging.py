"""Staging probe: N images of the C3 recipe written as .msft, then read back by
the per-file drop-in (load_dir) and by the threaded native bank loader."""
import os, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1512_06235_b200 import scenes, staging
from paper_1512_06235_b200.bank import HostBank

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
scene, _ = scenes.build("C3", n_cameras=n)
d = tempfile.mkdtemp()
for i, fs in scene.feature_sets.items():
    m = len(fs)
    head = np.array([0x5446534D, 1, i, fs.width, fs.height, m], "<u4").tobytes()   # "MSFT"
    rec = np.zeros((m, 144), np.uint8)
    f = np.empty((m, 4), "<f4")
    f[:, :2], f[:, 2], f[:, 3] = fs.xy, fs.scale, fs.orientation
    rec[:, :16] = f.view(np.uint8).reshape(m, 16)
    rec[:, 16:] = fs.descriptors
    open(os.path.join(d, f"{i:05d}.msft"), "wb").write(head + rec.tobytes())
mb = sum(os.path.getsize(os.path.join(d, x)) for x in os.listdir(d)) / 1e6
t0 = time.perf_counter(); store = staging.load_dir(d); t1 = time.perf_counter()
hb0 = HostBank(store.sets); t2 = time.perf_counter()
hb = staging.host_bank_from_dir(d); t3 = time.perf_counter()
assert np.array_equal(hb.desc.numpy(), hb0.desc.numpy())
print(f"{n} files {mb:.0f} MB: load_dir + HostBank {1e3*(t2-t0):.0f} ms; "
      f"native threaded bank {1e3*(t3-t2):.0f} ms ({mb/(t3-t2)/1e3:.2f} GB/s), {os.cpu_count()} threads")
