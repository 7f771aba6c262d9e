"""Per-tile timing of one config-2 render (diagnostic): where the step's time goes
across tiles, the tail, the slowest tiles.

    python -m paper_2602_03002_b200.build --out build/libmdrt_timing.so -D MDRT_TIMING
    python tools/tile_times.py [cfg2|cfg3]        # MDRT_TILE_ORDER=view|row as in the renderer
"""
import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
os.environ["MDRT_LIB"] = "build/libmdrt_timing.so"
import paper_2602_03002_b200 as md
from paper_2602_03002_b200 import synth, _native
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
w = synth.config(cfg)
C = len(w.cameras)
f32 = lambda x: np.asarray(x, np.float64).astype(np.float32).astype(np.float64)
bodies = [(nm, md.TriMesh(f32(m.vertices), m.faces, frame="body-local")) for nm, m in w.bodies]
scene = md.Scene(w.num_envs, bodies=bodies, cameras=w.cameras, terrain=md.TriMesh(f32(w.terrain.mesh.vertices), w.terrain.mesh.faces))
scene.set_camera_randomization(*md.sample_camera_offsets(md.CameraRandomization(seed=3), w.num_envs, C))
p, q = w.poses(0); scene.set_body_poses(p, q)
sens = md.SensorConfig()
flush = torch.empty(64 * 1024 * 1024, device="cuda")
for k in range(3):
    flush.fill_(k)
    md.render_pipeline(scene, sensor=sens, step=k)
torch.cuda.synchronize()
n = w.num_envs * C * 96
t0 = np.zeros(n, np.uint64); t1 = np.zeros(n, np.uint64)
L = _native.lib()
L.mdrt_debug_tile_times(t0.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), t1.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), n)
start = t0.min(); t0 = (t0 - start) / 1e3; t1 = (t1 - start) / 1e3
dur = t1 - t0
print("kernel span us", t1.max(), "tiles", n)
print("tile duration us: mean %.1f p50 %.1f p90 %.1f p99 %.1f max %.1f" % (dur.mean(), np.median(dur), np.percentile(dur, 90), np.percentile(dur, 99), dur.max()))
end = np.sort(t1)
print("last tile ends at", end[-1], "; 99.9% of tiles done by", end[int(0.999 * n)], "; 99% by", end[int(0.99 * n)])
first = t0 < 5
print("first wave (start < 5us):", first.sum(), "tiles, mean dur %.1f" % dur[first].mean(), "vs overall %.1f" % dur.mean())
# throughput per 100us window
hist, edges = np.histogram(t1, bins=np.arange(0, t1.max() + 100, 100))
print("tiles finished per 100us:", hist.tolist())
tpv = 96
txs = 16   # 4x8 tiles on 64x48: 16 x 6
views = w.num_envs * C
row_major = os.environ.get("MDRT_TILE_ORDER", "row") == "row"   # L2-resident configs default to row order
gws = np.arange(n)
if row_major:
    rows = gws // (views * txs); vv = (gws % (views * txs)) // txs; cols = gws % txs
else:
    vv = gws // tpv; rows = (gws % tpv) // txs; cols = (gws % tpv) % txs
print("order:", "tile-row-major" if row_major else "view-major")
order = np.argsort(-dur)[:30]
print("slowest tiles (us, view, tx, ty, start):")
for g in order:
    print("  %.1f view %d tx %d ty %d start %.0f" % (dur[g], vv[g], cols[g], rows[g], t0[g]))
print("mean duration by tile row:", [round(float(dur[rows == r].mean()), 1) for r in range(6)])
print("p99 duration by tile row:", [round(float(np.percentile(dur[rows == r], 99)), 1) for r in range(6)])
print("max duration by tile row:", [round(float(dur[rows == r].max()), 1) for r in range(6)])
print("p99 by tile column:", [round(float(np.percentile(dur[cols == c], 99)), 1) for c in range(16)])
print("max by tile column:", [round(float(dur[cols == c].max()), 1) for c in range(16)])
late = t0 > np.percentile(t1, 95)
print("tiles started in the last 5%% of the span: %d, mean dur %.1f, rows %s" % (late.sum(), dur[late].mean() if late.any() else 0, np.bincount(rows[late], minlength=6).tolist()))
