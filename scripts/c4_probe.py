"""C4 probe: generate the box-limited out-of-core city into tmpfs, then run
the session over the long street path and print per-frame paging stats."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2506_19415_b200 import scenegen
from paper_2506_19415_b200.scene_io import read_scene
from paper_2506_19415_b200.runtime import VmSession

lay = scenegen.C4
d = "/dev/shm/vmsplat_bench"
os.makedirs(d, exist_ok=True)
path = os.path.join(d, f"city_p{lay.n_pages}_s{lay.page_size}_l{lay.levels}_seed{lay.seed}.vms")
t = time.time()
if not os.path.exists(path):
    scenegen.write_city(path, lay)
print("gen s", round(time.time() - t, 1), "bytes", os.path.getsize(path), flush=True)
sc = read_scene(path, mmap_gaussians=True)
print("faces", len(sc.faces), "pages", sc.page_count, flush=True)
blocks = int(os.environ.get("BLOCKS", "24"))
buf = int(os.environ.get("BUF", "2048"))
stg = float(os.environ.get("STG", "160"))
traj = scenegen.street_path(lay, frames=120, blocks=blocks)
t = time.time()
s = VmSession(sc, buffer_pages=buf, staging_pages=stg, vis_scale=0.25, timing=True,
              upload_mode=int(os.environ.get("UPM", "2")))
print("session s", round(time.time() - t, 1), getattr(s.host, "kind", "?"), flush=True)
for f in range(traj.frame_count):
    t = time.time()
    _, st = s.render_frame(traj.frame_camera(f), f, out="device")
    if f % 4 == 0 or f < 8:
        print(f, {k: st[k] for k in ("required_pages", "resident_pages", "missing_pages",
                                     "planned_copies", "n_tris", "n_kept", "n_instances")},
              {k: round(st[k] * 1e3, 3) for k in ("time_visibility", "time_update", "time_copy",
                                                    "time_preprocess", "time_tiles", "time_blend",
                                                    "time_device_frame")},
              round((time.time() - t) * 1e3, 1), flush=True)
