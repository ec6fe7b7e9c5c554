"""Benchmark of the B200 fine-stage hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A step = geometry-aware matching of every densify pair of the C3 workload
(320-camera synthetic scene, 8k SIFT-like features/img,
3072x2304, ~5.4k visibility-filtered pairs) — BASELINE.json configs[2], the
config its "matched pairs/sec at 8k feats/img" metric is quoted on.  Pairs are
sharded round-robin over ranks (weak scaling), matches are gathered to rank 0
over NCCL.  Prints one JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "geometry-aware matched pairs/sec at 8k feats/img; localized images/sec"
UNIT = "pairs/s"
HBM_FALLBACK_GBS = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--cameras", type=int, default=320)
    p.add_argument("--cpu-pairs", type=int, default=0, help="CPU sample size (0 = auto)")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--chunk-pairs", type=int, default=0)
    p.add_argument("--segment-images", type=int, default=8,
                   help="e2e: bank images per staged upload range")
    p.add_argument("--e2e-resident", action="store_true",
                   help="e2e: upload + index the whole bank before matching (no staging)")
    p.add_argument("--no-localize", action="store_true")
    p.add_argument("--gather-chunks", type=int, default=4,
                   help="N > 1: pair chunks per rank whose rows go to rank 0 while the next "
                        "chunk computes")
    return p.parse_args()


# ---------------------------------------------------------------- workload --

def build_workload(n_cameras, with_snapshot=False):
    from paper_1512_06235_b200 import scenes

    scene, snap = scenes.build("C3", n_cameras=n_cameras)
    wl = scenes.pair_workload(scene, snap)
    ok = np.flatnonzero(wl.valid)
    if with_snapshot:
        return scene, wl, ok, snap
    return scene, wl, ok


def algorithmic_bytes(scene, wl, pairs, n_matches):
    """B_pair = 136|Q_u| + 136 n_t + 72 + 16|M_pair| (summed)."""
    nq = sum(len(wl.untracked[int(wl.q_img[k])]) for k in pairs)
    nt = sum(len(scene.feature_sets[int(wl.t_img[k])]) for k in pairs)
    return 136 * nq + 136 * nt + 72 * len(pairs) + 16 * int(n_matches)


# --------------------------------------------------------------- CPU legs ---

def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_oracle_rate(scene, wl, pairs, sample, seed=0):
    """Oracle port of guided_match_pair over a seeded pair sample, all host threads
    (ctypes releases the GIL).  Returns (pairs/s, cores, n_sample, seconds)."""
    from oracle import guided as og

    og.lib()
    rng = np.random.default_rng(seed)
    pick = rng.choice(len(pairs), size=min(sample, len(pairs)), replace=False)
    cores = cpu_cores()

    def one(j):
        k = int(pairs[j])
        q, t = int(wl.q_img[k]), int(wl.t_img[k])
        fq, ft = scene.feature_sets[q], scene.feature_sets[t]
        return len(og.guided_match(fq.xy, fq.descriptors, ft.xy, ft.descriptors, ft.width,
                                   ft.height, wl.F[k], wl.untracked[q])[0])

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=cores) as ex:
        list(ex.map(one, pick))
    dt = time.perf_counter() - t0
    return len(pick) / dt, cores, len(pick), dt


# ------------------------------------------------------------------ clocks --

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index=0):
        self.samples, self.stop, self.dev = [], threading.Event(), device_index
        self.ready = threading.Event()   # set at the first sample (NVML init is slow)
        self.nvml = False

    def _run_nvml(self):
        """NVML sampling every ~5 ms (the timed region is a few hundred ms)."""
        import pynvml as nv

        nv.nvmlInit()
        try:
            h = nv.nvmlDeviceGetHandleByIndex(self.dev)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
            self.nvml = True
            while not self.stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([str(sm), str(mx)] +
                                    ["Active" if r & b else "Not Active" for b in bits])
                self.ready.set()
                self.stop.wait(0.005)
        finally:
            nv.nvmlShutdown()

    def _run(self):
        try:
            self._run_nvml()
            return
        except Exception:
            self.samples.clear()
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.dev}",
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
                    self.ready.set()
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        # the sampler is running before the timed region starts: wait for its first
        # sample, then keep only what it records from here on (a timed region of a
        # few tens of ms otherwise ends before NVML has initialised)
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()
        self.ready.wait(timeout=5.0)
        if self.nvml:                    # 5-ms NVML samples: keep the timed region's only
            self.samples.clear()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def measured_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            j = json.load(f)
        return float(j.get("hbm_gbs", HBM_FALLBACK_GBS)), "measured"
    return HBM_FALLBACK_GBS, "fallback"


def ncu_unit_utilization(name):
    """Pipe / issue utilizations of a kernel from its committed ncu capture: which
    unit (if any) bounds it."""
    path = os.path.join(REPO, "profiles", name)
    if not os.path.exists(path):
        return None
    with open(path) as f:
        j = json.load(f)
    pick = {"issue_active_pct": "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
            "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "l2_sector_pct": "lts__t_sectors.sum.pct_of_peak_sustained_elapsed",
            "dram_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed"}
    out = {}
    for k, m in pick.items():
        v = j.get(m)
        if isinstance(v, dict):
            out[k] = round(float(v["value"]), 2)
    out["source"] = f"profiles/{name}"
    return out


def ncu_traffic_per_pair():
    """dram read+write bytes per pair of match_kernel from the committed ncu capture."""
    path = os.path.join(REPO, "profiles", "ncu_match_kernel.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        j = json.load(f)
    return j.get("dram_bytes_per_pair")


def ncu_traffic_source():
    """Where roofline.traffic comes from: the committed ncu capture's report name."""
    path = os.path.join(REPO, "profiles", "ncu_match_kernel.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        j = json.load(f)
    return (f"profiles/ncu_match_kernel.json: dram__bytes_read.sum + dram__bytes_write.sum "
            f"per pair from one ncu --set full capture ({j.get('report')}, "
            f"{j.get('pairs_per_launch', 0):.0f} pairs) of this build's match kernel on the C3 "
            f"step (tools/r2_measure_final.sh), scaled to this launch's pairs")


# --------------------------------------------------------------- main legs --

def kdtree_footnote(n_images=2, seed=0):
    """The reference's shipped default localization (DescriptorIndex picks its
    approximate kd-tree above 6,400 targets, descriptors.py:141-177) on a couple
    of C2 query images, when the unmodified reference is importable
    (baseline/_ref).  A footnote beside the exact oracle, not the baseline."""
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "msfm")):
        return {"unavailable": "baseline/_ref (pip install --target of the reference) absent"}
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        from msfm.features import FeatureSet as RFS, FeatureStore as RStore
        from msfm.localize import localize_image
        from msfm.matching import MatchGraph
        from msfm.model import Camera as RCam, FeatureRef as RRef, Model as RModel
    except Exception as exc:                       # a broken install must not end the run
        return {"unavailable": f"reference import failed: {exc}"}
    scene, snap, queries = build_localization()
    model = RModel(stage_tag="coarse")
    for i in snap.registered:
        c = scene.cameras[int(i)]
        model.attach_camera(RCam(K=c.K, R=c.R, t=c.t, image_id=int(i)))
    for p in range(len(snap.point_xyz)):
        lo, hi = snap.track_ptr[p], snap.track_ptr[p + 1]
        model.add_point(snap.point_xyz[p], [RRef(int(i), int(f)) for i, f in
                                            zip(snap.track_img[lo:hi], snap.track_fid[lo:hi])])
    sets = {}
    for i, fs in scene.feature_sets.items():
        sets[i] = RFS(image_id=fs.image_id, width=fs.width, height=fs.height, xy=fs.xy,
                      scale=fs.scale, orientation=fs.orientation, descriptors=fs.descriptors)
    store = RStore(sets)
    pick = [queries[j] for j in np.random.default_rng(seed).choice(len(queries), n_images,
                                                                   replace=False)]
    t0 = time.perf_counter()
    ok = 0
    for q in pick:
        try:
            r = localize_image(model, MatchGraph(), q, store, scene.cameras[q].K)
            ok += r.pose is not None
        except OverflowError:
            pass
    dt = time.perf_counter() - t0
    return {"value": len(pick) / dt, "unit": "images/s", "cores": 1, "kind": "reference",
            "sample": f"{len(pick)} C2 query images, msfm.localize.localize_image with the default "
                      f"DescriptorIndex (kd-tree above 6,400 targets), one thread, {dt:.1f} s",
            "localized": ok}


def run_reference(args, rank, world):
    """CPU reference arm: every timed step matches the FULL C3 pair list with the C
    restatement of guided_match_pair (oracle/guided_oracle.c) on all host threads
    — the b200 arm's config.  Warm-up steps run a 64-pair sample (they only page
    the code and the scene in; a full-list warm-up would add minutes and measure
    nothing)."""
    if rank != 0:
        return
    scene, wl, ok = build_workload(args.cameras)
    for i in range(args.warmup):
        cpu_oracle_rate(scene, wl, ok, 64, seed=i)
    times = []
    for i in range(args.steps):
        r, cores, n, dt = cpu_oracle_rate(scene, wl, ok, len(ok), seed=i)
        times.append(dt)
    ms = 1e3 * float(np.mean(times))
    v = len(ok) / (ms / 1e3)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "C3: geometry-aware matching of all densify pairs of a 320-camera "
                                   "synthetic scene, 8k feats/img, 3072x2304",
                       "pairs": int(len(ok)), "cameras": args.cameras,
                       "parallelism": f"{cores} host threads"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"all {len(ok)} C3 pairs every timed step "
                                       "(oracle/guided_oracle.c, the C restatement of "
                                       "msfm.guided.guided_match_pair); warm-up steps: 64 pairs"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "steps_ms": [round(1e3 * t, 1) for t in times]}
    if not args.no_localize:
        # the metric's second half: localized images/s of the CPU restatement on C2
        lscene, lsnap, queries = build_localization()
        lr, lcores, ln, ldt = cpu_localize_rate(lscene, lsnap, queries, len(queries))
        line["localization"] = {
            "metric": "localized images/sec", "value": lr, "unit": "images/s",
            "cpu_baseline": {"value": lr, "unit": "images/s", "cores": lcores, "kind": "port",
                             "sample": f"all {ln} C2 query images in {ldt:.1f}s (oracle/localize.py: "
                                       "exact direct 3D-2D + pnp_ransac restatement), one "
                                       "process per core"},
            "kdtree_default": kdtree_footnote()}
    print(json.dumps(line), flush=True)


def run_b200(args, rank, world):
    import torch
    import torch.distributed as dist

    from paper_1512_06235_b200 import _lib
    from paper_1512_06235_b200.bank import FeatureBank, HostBank
    from paper_1512_06235_b200.guided import (HostPairs, match_pairs, match_pairs_rows,
                                              match_pairs_rows_staged, prepare_pairs)

    from paper_1512_06235_b200.dist import ChunkGather, chunk_bounds

    dev = torch.device("cuda", 0 if os.environ.get("MSFM_BENCH_BACKEND") == "gloo"
                       else int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    scene, wl, ok, snap = build_workload(args.cameras, with_snapshot=True)
    mine = ok[rank::world]                     # round-robin over pair order (weak scaling)
    ql = [wl.untracked[int(wl.q_img[k])] for k in mine]
    host = HostBank(scene.feature_sets)
    bank = FeatureBank(host=host, device=dev)
    D = 8.0 * 1.25
    bank.grid(D)
    # N > 1: each rank's pairs in G chunks; chunk k's packed rows go to rank 0 (NCCL
    # point-to-point, capacity-sized buffers known to every rank) while chunk k+1
    # computes — the overlapped gather of SURVEY.md §8e
    G = max(1, args.gather_chunks) if world > 1 else 1
    qn = np.array([len(wl.untracked[int(wl.q_img[k])]) for k in ok], np.int64)
    caps, bounds_of = [], []
    for r in range(world):
        mr = np.arange(r, len(ok), world)
        b = chunk_bounds(len(mr), G)
        bounds_of.append(b)
        caps.append([int(qn[mr[b[k]:b[k + 1]]].sum()) for k in range(len(b) - 1)])
    bounds = bounds_of[rank]
    n_chunks = len(bounds) - 1
    chunk_inputs = [prepare_pairs(bank, wl.q_img[mine[bounds[k]:bounds[k + 1]]],
                                  wl.t_img[mine[bounds[k]:bounds[k + 1]]],
                                  wl.F[mine[bounds[k]:bounds[k + 1]]], ql[bounds[k]:bounds[k + 1]])
                    for k in range(n_chunks)]
    gathered = {}

    def step():
        gat = ChunkGather(world, rank, caps, dev) if world > 1 else None
        out = []
        for k in range(n_chunks):
            sl = slice(bounds[k], bounds[k + 1])
            res = match_pairs(bank, wl.q_img[mine[sl]], wl.t_img[mine[sl]], wl.F[mine[sl]], ql[sl],
                              device_inputs=chunk_inputs[k], chunk_pairs=args.chunk_pairs)
            out.append(res)
            if gat is not None:
                rows, cnt = res.packed_device()
                gat.put(k, rows, cnt)
        if gat is not None:
            got = gat.finish()
            if got is not None:
                gathered.clear()
                gathered.update(got)
        return out

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        res = step()
    torch.cuda.synchronize()
    n_matches_local = int(sum(int(r.count.sum().item()) for r in res))

    # ---- timed region: device-resident inputs -> matches (gathered on rank 0)
    l0 = _lib.launch_count()
    sampler = ClockSampler(dev.index)
    barrier(); torch.cuda.synchronize()
    with sampler:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            res = step()
        e1.record()
        torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    launches = (_lib.launch_count() - l0) // max(args.steps, 1)
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_pairs = len(ok)
    value = total_pairs * args.steps / (ms_max / 1e3)

    # ---- roofline: algorithmic bytes of this rank's pairs / match_kernel event time
    _lib.profile_enable(True)
    res = step()
    torch.cuda.synchronize()
    k_ms, k_n = _lib.profile_read("match_kernel")
    _lib.profile_enable(False)
    alg = algorithmic_bytes(scene, wl, mine, n_matches_local)
    peak, peak_kind = measured_peaks()
    achieved = alg / (k_ms / 1e3) / 1e9 if k_ms > 0 else 0.0
    step_ms = ms / args.steps
    tpp = ncu_traffic_per_pair()

    # ---- the stage's next step on the same matches: device track merge (densify.py:68-158)
    try:
        if world == 1:
            rows_all, _ = res[0].packed()
        else:
            # rank 0 holds every rank's rows (the last timed step's gather)
            from paper_1512_06235_b200.dist import merge_chunk_rows

            rows_all = None
            if rank == 0:
                index = {}
                for r in range(world):
                    mr = np.arange(r, len(ok), world)
                    b = bounds_of[r]
                    for k in range(len(b) - 1):
                        index[(r, k)] = mr[b[k]:b[k + 1]]
                rows_all = torch.from_numpy(merge_chunk_rows(gathered, index)).to(dev)
        merge = track_merge_leg(bank, wl, ok if world > 1 else mine, rows_all, snap, dev,
                                scene) if rows_all is not None else None
    except Exception as exc:                        # never lose the step's line over it
        merge = {"error": f"{type(exc).__name__}: {exc}"}

    # ---- e2e through the public API with host buffers (pinned H2D + D2H every step)
    torch.cuda.synchronize()
    e2e_ms = []
    h2d = d2h = 0
    pinned = torch.empty((max(int(sum(len(x) for x in ql)), 1), 4), dtype=torch.int32,
                         pin_memory=True)
    b2 = None
    hp = HostPairs(host, wl.q_img[mine], wl.t_img[mine], wl.F[mine], ql)   # pinned pair table
    for i in range(args.warmup + args.steps):
        barrier(); torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        if args.e2e_resident:
            b2 = FeatureBank(host=host, device=dev)
            b2.grid(D)
            inp = prepare_pairs(b2, wl.q_img[mine], wl.t_img[mine], wl.F[mine], ql)
            # matching with each chunk's packed rows copied to pinned memory while the
            # next chunk computes (msfm_guided_match_rows)
            rows = match_pairs_rows(b2, wl.q_img[mine], wl.t_img[mine], wl.F[mine], ql,
                                    device_inputs=inp, chunk_pairs=args.chunk_pairs,
                                    pinned=pinned)
        else:
            # the bank goes up range by range in the order the chunks need it, each
            # range indexed as it lands, chunk c starting once its ranges are ready;
            # packed rows of chunk c copied out while chunk c+1 computes
            rows, b2 = match_pairs_rows_staged(host, wl.q_img[mine], wl.t_img[mine],
                                               wl.F[mine], ql, device=dev,
                                               chunk_pairs=args.chunk_pairs, pinned=pinned,
                                               segment_images=args.segment_images, bank=b2,
                                               host_pairs=hp)
            inp = b2.pair_inputs
        a1.record()
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_ms.append(a0.elapsed_time(a1))
        h2d = host.nbytes + sum(int(x.numel() * x.element_size()) for x in inp[:5] + inp[6:])
        d2h = int(rows.nbytes + 16 * 6)   # packed 16-B rows + per-chunk (base, count)
    te = torch.tensor([float(np.mean(e2e_ms))], device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = total_pairs / (float(te.item()) / 1e3)

    # localization: query images sharded round-robin over the ranks (every rank runs)
    loc = run_localization(args, dev, world, rank) if not args.no_localize else None
    if rank != 0:
        return
    cpu = None
    # the CPU baseline is an N = 1 figure (rank 0 alone would share the host cores
    # with the other ranks' processes)
    if not args.no_cpu and world == 1:
        sample = args.cpu_pairs or max(8 * cpu_cores(), 96)
        r, cores, n, dt = cpu_oracle_rate(scene, wl, ok, sample)
        cpu = {"value": r, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{n} seeded-random C3 pairs in {dt:.1f}s (oracle/guided_oracle.c, the C "
                         f"restatement of msfm.guided.guided_match_pair), {cores} host threads"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": "C3: geometry-aware matching of all densify pairs of a 320-camera "
                               "synthetic scene, 8k feats/img, 3072x2304",
                   "pairs": int(total_pairs), "cameras": args.cameras,
                   "mean_queries_per_pair": float(np.mean([len(wl.untracked[int(wl.q_img[k])]) for k in ok])),
                   "parallelism": f"pairs round-robin over {world} GPU(s), no collective on "
                                  "the data path" + ("" if world == 1 else
                                  f"; each rank's rows go to rank 0 in {G} chunks over NCCL "
                                  "point-to-point, overlapping the next chunk's matching"),
                   "scaling_note": "C3's pair set sharded across ranks (BASELINE configs[2]); "
                                   "labelled weak per the sharded-independent-units rule",
                   "l2": "inputs larger than L2 (feature bank "
                         f"{host.nbytes / 1e6:.0f} MB > 126 MB); no explicit flush"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_kind": peak_kind,
                     "kernel": "match_kernel",
                     "traffic": (tpp * len(mine) / max(k_n, 1)) if tpp else None,
                     "traffic_source": ncu_traffic_source(),
                     "algorithmic_bytes_per_launch": alg / max(k_n, 1),
                     "launches": k_n, "kernel_ms_per_step": k_ms,
                     "step_frac": (alg / (step_ms / 1e3) / 1e9) / peak,
                     "units": ncu_unit_utilization("ncu_match_kernel.json")},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "steps_ms": [round(x, 2) for x in e2e_ms]},
        "gpu_launches": int(launches),
        "clocks": sampler.summary(),
        "matches_per_step": n_matches_local if world == 1 else None,
        "track_merge": merge,
    }
    if loc is not None:
        line["localization"] = loc
        line["coarse_graph"] = coarse_graph_leg(dev)
    print(json.dumps(line), flush=True)


def coarse_graph_leg(dev, n_cameras=40):
    """build_coarse_matchgraph (matching.py:208-249) on the C2 recipe's first
    n_cameras images at eta = 20 tiers: all pairs, hybrid matching on the tcgen05
    kNN, batched device F-RANSAC.  Wall clock (host orchestration included)."""
    import torch

    from paper_1512_06235_b200 import _lib, scenes
    from paper_1512_06235_b200.coarse import build_coarse_matchgraph

    scene, _ = scenes.build("C2", n_cameras=n_cameras)
    store = scene.store()
    store.apply_eta(20.0)
    build_coarse_matchgraph(store.sets, on_overflow="drop")
    torch.cuda.synchronize()
    _lib.profile_enable(True)
    t0 = time.perf_counter()
    g = build_coarse_matchgraph(store.sets, on_overflow="drop")
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    kern = {k: _lib.profile_read(k)[0] for k in ("knn_tc_kernel", "f_hyp_kernel",
                                                  "f_score_kernel", "f_refit_kernel")}
    _lib.profile_enable(False)
    P = n_cameras * (n_cameras - 1) // 2
    return {"metric": "coarse match-graph pairs/sec", "value": P / dt, "unit": "pairs/s",
            "workload": f"C2 recipe, {n_cameras} cameras, eta=20 tiers "
                        f"(~{int(np.mean([fs.coarse_count for fs in store.sets.values()]))} "
                        "features), all pairs",
            "pairs": P, "edges": len(g.edges), "overflow_pairs_dropped": len(g.overflow_pairs),
            "wall_ms": dt * 1e3, "kernel_ms": kern}


def track_merge_leg(bank, wl, pairs, rows, snap, dev, scene=None):
    """msfm_merge_tracks over the step's matches + the coarse tracks (bank nodes).
    ``rows``: device int32 (n, 4) packed match rows whose pair column indexes
    ``pairs``; with several ranks these are every rank's rows gathered on rank 0 —
    the gather of tracks of an N-GPU run."""
    import torch

    from paper_1512_06235_b200 import _lib
    from paper_1512_06235_b200.densify import merge_tracks_nodes

    n = int(rows.shape[0])
    qoff = torch.from_numpy(bank.offsets[bank.slots(wl.q_img[pairs])]).to(dev)
    toff = torch.from_numpy(bank.offsets[bank.slots(wl.t_img[pairs])]).to(dev)
    pk = rows[:, 0].long()
    u = (qoff[pk] + (rows[:, 1] & 0xFFFF).long()).to(torch.int32).contiguous()
    v = (toff[pk] + ((rows[:, 1] >> 16) & 0xFFFF).long()).to(torch.int32).contiguous()
    dist = rows[:, 2].contiguous().view(torch.float32)
    slot = np.array([bank.index_of[int(i)] for i in snap.track_img], np.int64)
    tnode = (bank.offsets[slot] + snap.track_fid).astype(np.int32)
    for _ in range(2):
        merge_tracks_nodes(bank, u, v, dist, snap.track_ptr, tnode)
    torch.cuda.synchronize()
    _lib.profile_enable(True)
    nodes, owners, offs = merge_tracks_nodes(bank, u, v, dist, snap.track_ptr, tnode)
    torch.cuda.synchronize()
    ms, _ = _lib.profile_read("merge_tracks")
    _lib.profile_enable(False)
    return {"what": "msfm_merge_tracks (densify.py:68-158) over the step's matches + the coarse "
                    "tracks, union-find over bank feature rows", "matches": int(n),
            "nodes": int(bank.n_total), "tracks": int(len(snap.track_ptr) - 1), "ms": ms,
            "edges_per_s": n / (ms / 1e3) if ms > 0 else None,
            "new_tracks": int((owners < 0).sum()), "extended_tracks": int((owners >= 0).sum()),
            "triangulation": triangulation_leg(scene, bank, nodes, owners, offs)}


def triangulation_leg(scene, bank, nodes, owners, offs):
    """Batched multi-view DLT triangulation (geometry.py:276-357) of the new tracks
    the merge produced: one msfm_triangulate_batch launch (C3 cameras = images)."""
    import torch

    from paper_1512_06235_b200 import _lib
    from paper_1512_06235_b200.triangulation import triangulate_batch

    if scene is None:
        return None
    new = np.flatnonzero(np.asarray(owners) < 0)
    seg = np.diff(offs)[new]
    ptr = np.zeros(len(new) + 1, np.int64)
    np.cumsum(seg, out=ptr[1:])
    sel = np.concatenate([np.arange(offs[s], offs[s + 1]) for s in new]) if len(new) else \
        np.zeros(0, np.int64)
    nd = np.asarray(nodes)[sel]
    slot = np.searchsorted(bank.offsets, nd, "right") - 1
    cam = np.asarray(bank.image_ids, np.int64)[slot].astype(np.int32)
    pix = bank.host.xy.numpy()[nd].astype(np.float64)
    K = np.stack([c.K for c in scene.cameras])
    R = np.stack([c.R for c in scene.cameras])
    t = np.stack([np.asarray(c.t).reshape(3) for c in scene.cameras])
    triangulate_batch(K, R, t, ptr, cam, pix)
    torch.cuda.synchronize()
    _lib.profile_enable(True)
    t0 = time.perf_counter()
    st, X, err = triangulate_batch(K, R, t, ptr, cam, pix)
    wall = time.perf_counter() - t0
    ms, _ = _lib.profile_read("tri_kernel")
    _lib.profile_enable(False)
    return {"what": "msfm_triangulate_batch over the merge's new tracks (DLT, Gauss-Newton, "
                    "depth / reprojection / angle gates)", "tracks": int(len(new)),
            "views": int(ptr[-1]), "kernel_ms": ms, "call_ms": wall * 1e3,
            "tracks_per_s": len(new) / (ms / 1e3) if ms > 0 else None,
            "accepted": int((st == 1).sum())}


# ------------------------------------------------------- localization leg ---

def build_localization():
    from paper_1512_06235_b200 import scenes

    scene, snap = scenes.build("C2")
    reg = set(int(i) for i in snap.registered)
    queries = [i for i in range(len(scene.cameras)) if i not in reg]
    return scene, snap, queries


def _cpu_localize_one(args):
    """oracle port: exact direct 3D-2D search + pnp_ransac restatement (one image)."""
    from oracle import localize as ol
    S, n, F, xyz, xy, K, seed = args
    corr = ol.direct_3d2d(np.arange(len(S)), S, n, F)
    if len(corr) <= 16:
        return "below_gate"
    try:
        r = ol.pnp_ransac(xyz[corr[:, 0]], xy[corr[:, 1]].astype(np.float64), K, seed=seed)
    except OverflowError:
        return "overflow"
    return "ok" if r is not None else "none"


def cpu_localize_rate(scene, snap, queries, sample, seed=0):
    import multiprocessing as mp

    from paper_1512_06235_b200 import scenes

    S, n = scenes.track_sums(scene, snap)
    rng = np.random.default_rng(seed)
    pick = rng.choice(len(queries), size=min(sample, len(queries)), replace=False)
    jobs = [(S, n, scene.feature_sets[queries[j]].descriptors, snap.point_xyz,
             scene.feature_sets[queries[j]].xy, scene.cameras[queries[j]].K, queries[j])
            for j in pick]
    cores = cpu_cores()
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(min(cores, len(jobs))) as pool:
        pool.map(_cpu_localize_one, jobs)
    dt = time.perf_counter() - t0
    return len(jobs) / dt, min(cores, len(jobs)), len(jobs), dt


def run_localization(args, dev, world=1, rank=0):
    """C2 localization leg.  With N ranks the 80 query images are sharded
    round-robin (localize.py:256-267: images are independent given the snapshot);
    the step time is the max over ranks; rank 0 returns the record."""
    import torch
    import torch.distributed as tdist

    from paper_1512_06235_b200 import _lib, scenes
    from paper_1512_06235_b200.bank import FeatureBank, HostBank
    from paper_1512_06235_b200.localize import (PointSet, direct_search, gather_pnp_inputs,
                                                knn2_tracks, knn2_tracks_staged, track_sums_device)
    from paper_1512_06235_b200.pnp import pnp_batch_flat

    scene, snap, all_queries = build_localization()
    queries = all_queries[rank::world]
    host = HostBank({q: scene.feature_sets[q] for q in queries})
    Ks = [scene.cameras[q].K for q in queries]
    # the coarse model's tracks as a CSR over a bank of the registered images: the
    # query points' exact track sums (K7, mean_descriptor localize.py:51-59) are
    # computed on the device inside every step
    reg = [int(i) for i in snap.registered]
    reg_host = HostBank({i: scene.feature_sets[i] for i in reg})
    reg_bank = FeatureBank(host=reg_host, device=dev)
    slot_of = {i: k for k, i in enumerate(reg_host.image_ids)}
    track_row = (reg_host.offsets[[slot_of[int(i)] for i in snap.track_img]]
                 + snap.track_fid).astype(np.int64)
    n = np.diff(snap.track_ptr).astype(np.int32)
    M = len(n)

    def points(rbank):
        dS, dn, dSS = track_sums_device(rbank, snap.track_ptr, track_row)
        return PointSet(S=None, n=n, ids=np.arange(M), dev=(dS, dn, dSS))

    def step(bank, pts, d_xyz, knn=None):
        # device-resident flat correspondences: image k owns [off[k], off[k+1]); the
        # gate of localize.py:203 (> 16) selects the images that go to PnP, and their
        # 3D-2D pairs are gathered on the device
        corr = direct_search(bank, pts, queries, to_host=False, knn=knn)
        X, uv, toff, todo = gather_pnp_inputs(bank, corr, queries, d_xyz)
        res = pnp_batch_flat(X, uv, toff, [Ks[k] for k in todo], [queries[k] for k in todo],
                             device=dev)
        return toff, res

    bank = FeatureBank(host=host, device=dev)
    d_xyz = torch.from_numpy(snap.point_xyz).to(dev)
    for _ in range(args.warmup):
        corrs, res = step(bank, points(reg_bank), d_xyz)
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        corrs, res = step(bank, points(reg_bank), d_xyz)
    e1.record()
    torch.cuda.synchronize()
    tt = torch.tensor([e0.elapsed_time(e1) / 1e3 / args.steps], device=dev)
    if world > 1:
        tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
    dt = float(tt.item())
    status = {}
    for r in res:
        status[r.status] = status.get(r.status, 0) + 1
    # roofline of the kNN kernel: 2 planes x 2*M*N*128 int8 ops vs 2x measured bf16 (int8 rate)
    pts = points(reg_bank)
    _lib.profile_enable(True)
    knn2_tracks(bank, pts, queries)
    torch.cuda.synchronize()
    k_ms, k_n = _lib.profile_read("knn_tc_kernel")
    _lib.profile_enable(False)
    N_feat = int(sum(len(scene.feature_sets[q]) for q in queries))
    ops_alg = 2.0 * M * N_feat * 128
    ops_hw = 2.0 * ops_alg
    peak, peak_kind = None, None
    extra = os.path.join(REPO, "profiles", "measured_peaks_extra.json")
    if os.path.exists(extra):
        with open(extra) as f:
            peak = float(json.load(f).get("int8_dense_tops", 0)) or None
        peak_kind = "measured int8 dense tcgen05 burst (profiles/measured_peaks_extra.json)"
    if peak is None:
        path = os.path.join(REPO, "MEASURED_PEAKS.json")
        if os.path.exists(path):
            with open(path) as f:
                peak = 2.0 * float(json.load(f).get("bf16_tflops", 1590.0))
        peak = peak or 2.0 * 1590.0
        peak_kind = "2x measured bf16 (int8 dense rate)"
    ach = ops_hw / (k_ms / 1e3) / 1e12 if k_ms > 0 else 0.0
    # e2e: features + points H2D every step
    e2e = []
    b2 = FeatureBank(host=host, device=dev, staged=True)   # device buffers reused per step
    pin_xyz = torch.from_numpy(snap.point_xyz).pin_memory()
    for i in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        # the registered images' rows go up and their tracks are summed on the device;
        # the query bank goes up in eight ranges, each range's kNN starting as it lands
        reg_bank.refill()
        p2 = points(reg_bank)
        knn = knn2_tracks_staged(b2, p2, queries, p2.dev)
        step(b2, p2, pin_xyz.to(dev, non_blocking=True), knn=knn)
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e.append(time.perf_counter() - t1)
    te = torch.tensor([float(np.mean(e2e))], device=dev)
    cnts = torch.tensor([status.get(k, 0) for k in ("ok", "none", "overflow", "insufficient")],
                        device=dev, dtype=torch.int64)
    if world > 1:
        tdist.all_reduce(te, op=tdist.ReduceOp.MAX)
        tdist.all_reduce(cnts)
    e2e_s = float(te.item())
    status = {k: int(v) for k, v in zip(("ok", "none", "overflow", "insufficient"), cnts.tolist()) if v}
    if rank != 0:
        return None
    out = {"metric": "localized images/sec",
           "workload": f"C2: 100-camera scene, 8k feats/img, 20% coarse model (M={M} points), "
                       f"{len(all_queries)} query images: exact kNN + ratio + seeded PnP-RANSAC"
                       + ("" if world == 1 else f", images round-robin over {world} GPUs"),
           "value": len(all_queries) / dt, "unit": "images/s",
           "ms_per_step": dt * 1e3, "status_counts": status,
           "e2e": {"value": len(all_queries) / e2e_s, "unit": "images/s",
                   "h2d_bytes_per_step": int(host.nbytes + reg_host.nbytes + 8 * (M + 1)
                                             + 8 * len(track_row) + 24 * M),
                   "d2h_bytes_per_step": int(4 * len(queries) + 13 * 8 * len(res) +
                                             sum(r.mask.nbytes for r in res if r.mask is not None))},
           "roofline": {"bound": "tensor", "kernel": "knn_tc_kernel", "achieved": ach,
                        "peak": peak, "unit": "TOPS (int8)", "frac": ach / peak,
                        "peak_kind": peak_kind,
                        "ops_per_launch_hw": ops_hw, "ops_per_launch_alg": ops_alg,
                        "kernel_ms": k_ms, "alg_frac": (ops_alg / (k_ms / 1e3) / 1e12) / peak
                        if k_ms > 0 else 0.0,
                        "units": ncu_unit_utilization("ncu_knn_tc_kernel.json")}}
    out["n_gpus"] = world
    out["roofline"]["note"] = "rank 0's image shard" if world > 1 else None
    if not args.no_cpu and world == 1:
        r, cores, ns, cdt = cpu_localize_rate(scene, snap, queries, max(cpu_cores(), 8))
        out["cpu_baseline"] = {"value": r, "unit": "images/s", "cores": cores, "kind": "port",
                               "sample": f"{ns} query images in {cdt:.1f}s (oracle/localize.py: "
                                         "exact direct 3D-2D + pnp_ransac restatement), one "
                                         "process per core"}
    return out


def relaunch(args):
    """--gpus N > 1 outside torchrun: start N ranks (one per GPU) with
    torch.distributed.run on this node and return its exit code."""
    import socket

    if args.impl == "b200":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus and os.environ.get("MSFM_BENCH_BACKEND") != "gloo":
            print(json.dumps({"error": f"--gpus {args.gpus} but only {have} CUDA device(s) visible"}),
                  flush=True)
            return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if args.impl == "b200" else "gloo"
        # rehearsal of the N-rank code path on one GPU (NCCL refuses two ranks on
        # one device): every rank on cuda:0, host collectives over gloo
        backend = os.environ.get("MSFM_BENCH_BACKEND", backend)
        dist.init_process_group(backend=backend)
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        else:
            run_b200(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
