/*
 * vmsplat_b200 — C ABI of the B200-native per-frame VM/LOD splat path.
 *
 * Drop-in boundary for the reference package `vmsplat` (arXiv 2506.19415
 * restatement).  The reference binds its native code through Python: the
 * `vmsplat.kernels` wrappers (pkg/src/vmsplat/kernels/__init__.py:24-51)
 * call the Cython core (pkg/src/vmsplat/kernels/_core.pyx), and
 * `VmSession.render_frame` (pkg/src/vmsplat/runtime.py:436-489) strings the
 * per-frame stages together in NumPy.  Every entry point below replaces one
 * of those, as cited per function; the ctypes binding that plays the role of
 * the reference's Cython module lives in paper_2506_19415_b200/_lib.py and
 * is reproduced in INTEGRATION.md.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Pointers marked [dev] are device (or
 *    device-mapped pinned host) memory; [host] are host memory.
 *  - `stream` is a cudaStream_t passed as void*; NULL = legacy stream.
 *  - Every int32_t-returning call returns a VMS_* status; vms_last_error()
 *    gives the thread-local message of the last failure.  Status codes map
 *    onto the reference's exceptions (pkg/src/vmsplat/errors.py:1-26):
 *    VMS_ERR_INVARIANT / VMS_ERR_RANGE -> InvariantViolation,
 *    VMS_ERR_INVALID -> ValueError/DataError, VMS_ERR_CUDA -> RuntimeError.
 *  - No hot-path allocation: callers size workspaces with the *_bytes
 *    queries and own every buffer (kernels hold no state).
 *  - Results are bit-exact with the reference for every integer/index output
 *    (page-ID images, required lists, plans, sort orders).  Images: exact
 *    mode (the default; FP64 blend arithmetic like the reference) is within
 *    1e-5 max-abs of the reference; fast mode (opt-in, certified FP32 blend)
 *    is within 1e-3 max-abs: each pixel carries a running bound on its FP32
 *    transmittance and colour error, and every pixel whose 1/255 stop
 *    decision or colour (> 9e-4) the bound cannot certify is re-blended with
 *    the exact FP64 arithmetic (tests/test_gpu_parity.py checks both).
 */
#ifndef VMSPLAT_B200_H
#define VMSPLAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VMS_OK 0
#define VMS_ERR_INVALID 1
#define VMS_ERR_RANGE 2
#define VMS_ERR_CUDA 3
#define VMS_ERR_NOMEM 4
#define VMS_ERR_INVARIANT 5

#define VMS_ABI_VERSION 1

/* Camera for a kernel launch: render.Camera (pkg/src/vmsplat/render.py:47-101)
 * reduced to the numbers the kernels use.  rot = quat_to_matrix(orientation),
 * row-major, view = (p - pos) @ rot.  dot_mode selects the FP64 dot order
 * matching the host BLAS (0 = fused fma chain, 1 = unfused), probed once per
 * session. */
typedef struct vms_camera {
  double pos[3];
  double rot[9];
  double focal;
  double half_w;
  double half_h;
  double near;
  int32_t width;
  int32_t height;
  int32_t dot_mode;
  int32_t pad_;
} vms_camera;

/* LOD thresholds (runtime.LodController.thresholds, runtime.py:99-121). */
typedef struct vms_lod {
  double thresholds[8];
  int32_t count;
  int32_t pad_;
} vms_lod;

/* Required-page list (runtime.RequiredList, runtime.py:46-60) in compacted
 * form, ascending page id, written by the GPU into [dev]-mapped pinned host
 * memory.  meta[0] = clipped triangles, meta[1] = required pages,
 * meta[2] = largest out-of-range page id seen (0 = none). */
typedef struct vms_required_out {
  uint32_t* pid;
  uint32_t* enc;
  uint8_t* direct;
  uint8_t* level;
  uint32_t* meta;
} vms_required_out;

typedef struct vms_vis_args {
  vms_camera cam;               /* the visibility camera (camera.scaled(vis_scale)) */
  const double* verts;          /* [dev] (nv, 3) f64 proxy-mesh vertices */
  const int32_t* faces;         /* [dev] (nf, 3) */
  const uint32_t* face_page;    /* [dev] (nf,) page id per face, 0 = occluder */
  uint32_t n_faces;
  uint32_t page_count;
  const uint32_t* link_off;     /* [dev] (P + 1,) CSR offsets (scene_io.py:163-165) */
  const uint32_t* link_tgt;     /* [dev] link targets */
  vms_lod lod;
  uint32_t* id_image;           /* [dev] optional (h, w) page-ID image */
  double* invz_image;           /* [dev] optional (h, w) 1/z image */
  uint32_t* depth_out;          /* [dev] optional (P + 1,) encoded depths after links */
  uint8_t* direct_out;          /* [dev] optional (P + 1,) direct flags */
  vms_required_out out;
  void* workspace;              /* [dev] vms_visibility_workspace_bytes() */
} vms_vis_args;

/* A run of <= 128 resident records: device-pool rows [row, row + count)
 * carry gather indices [gather, gather + count) (runtime.gather_resident,
 * runtime.py:377-390, without the gather copy). */
typedef struct vms_chunk {
  uint32_t row;
  uint32_t gather;
  uint32_t count;
  uint32_t pad_;
} vms_chunk;

typedef struct vms_render_args {
  vms_camera cam;
  const float* pool;            /* [dev] (rows, 59) f32 record pool */
  const vms_chunk* chunks;      /* [dev] chunk table */
  uint32_t n_chunks;
  uint32_t n_splats;            /* gather indices in use (resident records) */
  uint32_t n_cap;               /* workspace splat capacity */
  uint32_t m_cap;               /* workspace tile-instance capacity */
  float* image;                 /* [dev] (h, w, 3) f32 output */
  int32_t accumulate;           /* 1: blend over image's current content */
  int32_t exact;                /* 1: FP64 blend (reference arithmetic) */
  uint32_t* counters_out;       /* [host pinned] optional: n_kept, n_inst, overflow */
  void* workspace;              /* [dev] vms_render_workspace_bytes() */
  void* events[4];              /* optional cudaEvent_t, recorded after: preprocess,
                                   depth sort, tile sort (blend start), blend */
} vms_render_args;

/* One planned page copy in bytes (runtime.execute_copies, runtime.py:362-374). */
typedef struct vms_copy {
  uint64_t src_offset;
  uint64_t dst_offset;
  uint64_t nbytes;
} vms_copy;

typedef struct vms_pagetable vms_pagetable;

/* ---- library --------------------------------------------------------- */
const char* vms_last_error(void);
int32_t vms_abi_version(void);
/* Edge (pixels) of the square blend tiles: 32, or 16 with VMSPLAT_TILE=16. */
int32_t vms_tile_size(void);
/* 1 if `ptr` is page-locked host memory the device can address (zero-copy
 * target), 0 otherwise. */
int32_t vms_host_accessible(const void* ptr);
/* Page-lock (and map into the device address space) an existing host range,
 * e.g. the read-only memory map of a .vms file's record section
 * (scene_io.py:318-321 read_scene(mmap)), so several sessions - and several
 * processes, one per GPU, mapping the same file - stream pages from ONE
 * host-resident copy of the scene instead of each holding a private pinned
 * copy.  The range is widened to whole pages; *base_out receives the
 * registered base for vms_host_unregister.  read_only adds
 * cudaHostRegisterReadOnly (required for PROT_READ mappings). */
int32_t vms_host_register(const void* ptr, uint64_t bytes, int32_t read_only, void** base_out);
int32_t vms_host_unregister(void* base);

/* Per-launch device timing for profiling runs: when enabled every kernel
 * launch records a CUDA event; the report (CSV "kernel,count,total_us")
 * attributes consecutive event deltas on a stream to kernels.  Returns the
 * report length; buf may be NULL to query it. */
int32_t vms_profile_enable(int32_t on);
int64_t vms_profile_report(char* buf, int64_t len);
/* Profiling: when dev_ptr is non-NULL every blend CTA writes {start ns, end
 * ns, SM id, (list length << 32) | tile} (4 x u64) at dev_ptr[4 * block]. */
int32_t vms_debug_blend_trace(void* dev_ptr);
/* The exact blend's table-driven FP64 exp(x), x in [-700, 0], evaluated on
 * [dev] x -> [dev] out (accuracy test against libm; not on the hot path). */
int32_t vms_debug_exp(const double* x, int64_t n, double* out, void* stream);
/* Certified fast blend (exact = 0): on != 0 flags every pixel, so the whole
 * image is re-blended by the FP64 repair kernel (tests: must equal exact
 * mode). */
int32_t vms_debug_cert_all(int32_t on);
/* Exact blend: per-pixel splat walks for groups of small splats (on = 1,
 * the default; VMSPLAT_LANE_LISTS) when they save more than margin steps -
 * for same-process A/B and identity tests (synchronises the device). */
int32_t vms_debug_lane_lists(int32_t on, int32_t margin);

/* ---- kernel-level drop-ins (pkg/src/vmsplat/kernels/__init__.py) ------ */

/* composite_splats (kernels/__init__.py:24-33, _core.pyx:24-78): blend n
 * caller-ordered splats into image (h, w, 3) f32 in place.  n_instances is
 * the tile-instance capacity (sum over splats of the blend tiles their
 * clamped box touches); an undersized capacity still gives the exact image,
 * blended from the ordered splat list instead of per-tile lists (slower). */
size_t vms_composite_workspace_bytes(int64_t n, int64_t n_instances, int32_t h, int32_t w);
int32_t vms_composite_splats(const float* centers, const float* conics, const float* colors,
                             const float* alphas, const int32_t* bounds, int64_t n,
                             int64_t n_instances, float* image, int32_t h, int32_t w,
                             int32_t exact, void* workspace, size_t workspace_bytes,
                             void* stream);

/* rasterize_triangles (kernels/__init__.py:36-43, _core.pyx:81-159): tris
 * (n, 3, 3) f64 of (x, y, 1/z); depth-tested in place into id_image / invz. */
size_t vms_rasterize_workspace_bytes(int64_t n);
int32_t vms_rasterize_triangles(const double* tris, const uint32_t* ids, int64_t n,
                                uint32_t* id_image, double* invz_image, int32_t h, int32_t w,
                                void* workspace, size_t workspace_bytes, void* stream);

/* radix_sort_pairs (kernels/__init__.py:46-51, _core.pyx:162-202): stable
 * ascending sort of u32 keys carrying an i64 payload, in place. */
size_t vms_radix_workspace_bytes(int64_t n);
int32_t vms_radix_sort_pairs(uint32_t* keys, int64_t* values, int64_t n, void* workspace,
                             size_t workspace_bytes, void* stream);

/* bvh_nearest_points (kernels/__init__.py:54-63, _core.pyx:279-334): nearest
 * face per query point over the flat median-split BVH of mesh/geometry.py
 * FaceBvh (bounds (n_nodes, 6) f64 lo|hi, children (n_nodes, 2) i32 with
 * (-1, -1) for leaves, ranges (n_nodes, 2) i32 half-open spans of tri_order,
 * tri_verts (n_faces, 3, 3) f64).  out_face i64 (lowest face index on
 * distance ties), out_dist f64 - bit-identical to the reference.  All
 * pointers are device memory; *overflow (device i32) is set when a query
 * needs more than the reference's 128-entry traversal stack (the reference
 * raises RuntimeError; so does the Python wrapper). */
int32_t vms_bvh_nearest_points(const double* points, int64_t n_points, const double* bounds,
                               const int32_t* children, const int32_t* ranges, int64_t n_nodes,
                               const int32_t* tri_order, const double* tri_verts,
                               int64_t n_faces, int64_t* out_face, double* out_dist,
                               int32_t* overflow, void* stream);

/* Camera.world_to_view (render.py:79-81) on the device; also the probe that
 * picks dot_mode against the host BLAS. out (n, 3) f64. */
int32_t vms_world_to_view(const double* points, int64_t n, const vms_camera* cam, double* out,
                          void* stream);

/* project_records + compute_keys (render.py:138-220) over a contiguous [dev]
 * (n, 59) f32 record array, one row per output index.  keys[i] = IEEE bits of
 * f32 view z for live rows (opacity > 0, z > near), 0xFFFFFFFF otherwise.
 * centers f64 (n,2), conics f64 (n,3), colors f32 (n,3), bounds i32 (n,4)
 * half-open, kept u8 (n,): written together (all null to skip); rows with
 * kept == 0 leave the geometry outputs untouched. */
int32_t vms_project_records(const float* records, int64_t n, const vms_camera* cam,
                            double* centers, double* conics, float* colors, int32_t* bounds,
                            uint8_t* kept, uint32_t* keys, void* stream);

/* evaluate_sh (render.py:104-135): coeffs (n, 16, 3) f64, dirs (n, 3) f64 unit
 * vectors -> out (n, 3) f64 = max(0, 0.5 + sum). */
int32_t vms_evaluate_sh(const double* coeffs, const double* dirs, int64_t n, double* out,
                        void* stream);

/* ---- per-frame stages (runtime.VmSession.render_frame) ----------------- */

/* render_visibility + reduce_visibility + select_lod (render.py:279-307,
 * runtime.py:70-96,129-132): subsystems [1] and [2]. */
size_t vms_visibility_workspace_bytes(uint32_t n_faces, uint32_t page_count);
int32_t vms_visibility(const vms_vis_args* args, void* stream);

/* reduce_visibility (runtime.py:70-96) over a given page-ID image and f64
 * depth image: depths_out (P + 1,) encoded nearest depth after the one-hop
 * link pass, direct_out (P + 1,) u8, *bad_id_out = largest id > P (0 = ok;
 * the caller raises InvariantViolation).  workspace >= 4 * (P + 1) bytes. */
int32_t vms_reduce_visibility(const uint32_t* page_image, const double* depth_image,
                              int64_t n_pixels, uint32_t page_count, const uint32_t* link_off,
                              const uint32_t* link_tgt, uint32_t* depths_out, uint8_t* direct_out,
                              uint32_t* bad_id_out, void* workspace, size_t workspace_bytes,
                              void* stream);

/* execute_copies (runtime.py:362-374): subsystem [3] data movement.
 * mode 0: copy engines, one cudaMemcpyAsync per run of copies adjacent in
 * both source and destination (pinned host source; copies in host memory);
 * mode 1: one gather kernel reading mapped pinned host memory (copies in
 * [dev]-accessible memory; occupies SMs while it waits on PCIe). */
int32_t vms_upload_pages(const vms_copy* copies, int64_t n, const void* host_base,
                         void* dev_base, int32_t mode, void* stream);

/* gather_resident + depth_order + composite_ordered (runtime.py:377-390,
 * render.py:235-248): subsystems [4], [5], [6]. */
size_t vms_render_workspace_bytes(uint32_t n_cap, uint32_t m_cap, int32_t width,
                                  int32_t height);
int32_t vms_render(const vms_render_args* args, void* stream);

/* ---- page table (runtime.PageTable / update_page_table, runtime.py:161-346)
 * Host C++ with O(log n) allocation; exact reference semantics. */
vms_pagetable* vms_pt_create(int64_t capacity);
void vms_pt_destroy(vms_pagetable* pt);
int32_t vms_pt_update(vms_pagetable* pt, const uint32_t* pid, const uint32_t* enc,
                      const uint8_t* direct, const uint8_t* level, int64_t n, int64_t frame,
                      double budget, uint32_t* plan_pid, uint8_t* plan_level,
                      int32_t* plan_entry, int32_t* plan_slot, int64_t plan_cap,
                      int64_t* n_plan, int64_t* missing);
int64_t vms_pt_capacity(const vms_pagetable* pt);
int64_t vms_pt_occupied(const vms_pagetable* pt);
int64_t vms_pt_resident_count(const vms_pagetable* pt);
int32_t vms_pt_resident(const vms_pagetable* pt, uint32_t* pid, int32_t* entry, int32_t* slot,
                        int64_t cap);
int32_t vms_pt_entries(const vms_pagetable* pt, int32_t* level, int64_t* last_used,
                       uint32_t* slots, int32_t max_slots);
int32_t vms_pt_resident_counts(const vms_pagetable* pt, int64_t* counts, int32_t levels);
int32_t vms_pt_check(const vms_pagetable* pt);
int64_t vms_pt_chunks(const vms_pagetable* pt, int64_t page_size, vms_chunk* out, int64_t cap,
                      int64_t* n_records);

/* ---- whole frames: VmSession (runtime.py:393-489) -------------------------
 * One host call per frame: visibility -> (event sync) -> page table ->
 * uploads on a side stream -> chunk table -> render.  The session owns the
 * page table, two CUDA events/streams and small pinned buffers; the caller
 * owns the big buffers (pool, workspaces, the pinned host scene). */
typedef struct vms_session vms_session;

typedef struct vms_session_desc {
  const float* host_records;    /* the GAUS section, all levels: [dev-mapped pinned] for
                                   upload_mode 0/1; any host memory (e.g. the mmap of the
                                   .vms file) for upload_mode 2 */
  uint64_t host_rows;
  uint32_t page_size;
  uint32_t lod_levels;          /* levels stored in the scene */
  uint32_t page_counts[16];     /* pages per level (scene_io.py:144-157) */
  uint32_t page_count;          /* level-0 pages P */
  uint32_t n_faces;
  const double* verts;          /* [dev] */
  const int32_t* faces;         /* [dev] */
  const uint32_t* face_page;    /* [dev] */
  const uint32_t* link_off;     /* [dev] (P + 1,) - all zero when links are disabled */
  const uint32_t* link_tgt;     /* [dev] */
  float* pool;                  /* [dev] capacity * page_size rows of 59 f32 */
  uint32_t capacity;            /* buffer_pages */
  uint32_t m_cap;               /* tile-instance capacity of render_ws */
  void* vis_ws;                 /* [dev] vms_visibility_workspace_bytes(n_faces, P) */
  void* render_ws;              /* [dev] vms_session_render_ws_bytes(...) */
  uint64_t render_ws_bytes;
  int32_t width;                /* render resolution render_ws is sized for */
  int32_t height;
  int32_t exact;                /* 1: FP64 blend */
  int32_t upload_mode;          /* 0/1: see vms_upload_pages; 2: streaming - planned rows are
                                   gathered by host threads into a page-locked bounce buffer,
                                   one cudaMemcpyAsync per frame */
  int32_t host_fd;              /* upload_mode 2: >= 0 -> the rows are read with pread() from
                                   this file (the .vms) at host_fd_offset + row * 236 instead
                                   of being copied out of host_records (no page faults on a
                                   fresh mapping); -1 -> copy from host_records */
  uint64_t host_fd_offset;      /* byte offset of the record section in host_fd */
  int32_t device_table;         /* 1: the page table lives on the device (vms_dpt, SURVEY
                                   8(f) F2) - updated by a kernel right after the visibility
                                   pass, the host only issues the planned copies; needs
                                   capacity <= 8192 and lod_levels <= 6 */
  int32_t pad_;
} vms_session_desc;

typedef struct vms_frame_args {
  vms_camera cam;               /* render camera */
  vms_camera vis_cam;           /* camera.scaled(vis_scale) */
  vms_lod lod;                  /* controller thresholds before this frame's adaptation */
  int64_t frame;
  double budget;                /* staging_pages */
  float* image;                 /* [dev] (h, w, 3); may be device-accessible pinned host
                                   memory (zero-copy: the blend writes over PCIe) */
  float* host_image;            /* [host pinned] optional: D2H + sync at the end */
  int32_t timing;               /* 1: stage CUDA events + sync at the end */
  int32_t sync;                 /* 1: return only once the frame is complete */
} vms_frame_args;

typedef struct vms_frame_stats {
  uint32_t required;            /* len(required_ids) */
  uint32_t resident;            /* len(table.resident) */
  uint32_t planned;             /* len(plan) */
  uint32_t missing;
  uint64_t bytes_copied;
  uint32_t occupied_entries;    /* usage = occupied_entries / capacity */
  uint32_t capacity;
  uint32_t n_tris, n_chunks, n_res;
  uint32_t n_kept, n_inst, overflow, n_need;  /* valid when the call synchronised */
  uint32_t pad_;
  int64_t resident_per_level[16];
  float ms_vis, ms_copy, ms_preprocess, ms_sort, ms_tiles, ms_blend, ms_frame;
  float ms_host_gather;         /* upload_mode 2: host time reading the planned rows */
  double host_update_s;
} vms_frame_stats;

size_t vms_session_render_ws_bytes(uint32_t capacity, uint32_t page_size, uint32_t m_cap,
                                   int32_t width, int32_t height);
vms_session* vms_session_create(const vms_session_desc* desc);
void vms_session_destroy(vms_session* s);
vms_pagetable* vms_session_table(vms_session* s);
int32_t vms_session_set_render_ws(vms_session* s, void* ws, uint64_t bytes, uint32_t m_cap,
                                  int32_t width, int32_t height);
/* One frame (runtime.py:436-489).  Returns once the frame is enqueued: the
 * visibility pass and the host page table are done, the render is in flight
 * on `stream` (replayed from a CUDA graph).  With host_image or timing set the
 * call also waits for the render and fills the device counters.  A frame
 * whose tile instances overflow the buffer is still blended exactly (through
 * the depth-sorted splat list, slower); the session grows the buffer for the
 * frames after it. */
int32_t vms_session_frame(vms_session* s, const vms_frame_args* args, vms_frame_stats* stats,
                          void* stream);
/* Wait for the last frame (back = 0) or one of the frames before it (back <
 * vms_session_slots): with a device-accessible host image and sync = 0,
 * vms_session_frame returns as soon as the frame is enqueued and this is how
 * the caller learns that the image is complete. */
int32_t vms_session_wait(vms_session* s, int32_t back);
/* Frames a session keeps in flight (2..8, VMSPLAT_SLOTS, default 4):
 * vms_session_frame for frame i waits for frame i - slots. */
int32_t vms_session_slots(const vms_session* s);
/* Allocate the render workspaces of every frame slot for width x height now
 * (a session otherwise allocates them at its first frame; nothing else
 * changes - the page cache stays cold). */
int32_t vms_session_prepare(vms_session* s, int32_t width, int32_t height);
/* Wait for the last frame; out4 = its n_kept, n_inst, overflow, n_need. */
int32_t vms_session_counters(vms_session* s, uint32_t* out4, void* stream);

/* ---- device-resident page table ------------------------- */

/* Opaque device page table (csrc/dpt.cu): the state of runtime.PageTable
 * (runtime.py:161-291) in device memory; capacity <= 8192 entries, levels
 * <= 6.  Not thread-safe; one stream at a time. */
typedef struct vms_dpt vms_dpt;

typedef struct vms_dpt_frame {  /* [dev] per-frame inputs of the update */
  int64_t frame;
  double budget;                /* staging budget in level-0 pages */
} vms_dpt_frame;

typedef struct vms_dpt_stats {  /* [dev or mapped host] per-frame outputs */
  uint32_t n_req, n_plan, missing, resident, occupied, bad, plan_overflow;
  uint32_t n_chunks, n_records, pad_;
  uint32_t resident_per_level[16];
} vms_dpt_stats;

vms_dpt* vms_dpt_create(int32_t capacity, int32_t page_count, int32_t levels);
/* The device table of a session created with device_table = 1 (else NULL). */
vms_dpt* vms_session_dpt(vms_session* s);
/* Pixels the last frame's certified fast blend re-blended in FP64
 * (synchronises the device; exact = 0 sessions). */
int32_t vms_session_cert_count(vms_session* s, uint32_t* out);
void vms_dpt_destroy(vms_dpt* d);
size_t vms_dpt_smem_bytes(const vms_dpt* d);
/* update_page_table (runtime.py:294-346) on the device: the required list
 * (ascending page id, [dev] arrays as reduce_visibility + select_lod produce
 * them, *n_req [dev]) -> the copy plan (pid, level, entry, slot) in the
 * reference's order, stats.  Bit-identical plans, residency, LRU stamps and
 * missing counts to the reference (and to vms_pt_update).  Graph-capturable. */
int32_t vms_dpt_update(vms_dpt* d, const uint32_t* pid, const uint32_t* enc,
                       const uint8_t* direct, const uint8_t* level, const uint32_t* n_req,
                       const vms_dpt_frame* frame, uint32_t* plan_pid, uint8_t* plan_level,
                       int32_t* plan_entry, int32_t* plan_slot, int64_t plan_cap,
                       vms_dpt_stats* stats, void* stream);
/* gather_resident's order (runtime.py:377-390) as <= 128-record chunks
 * {pool row, gather index, count} of every resident page, ascending page id,
 * into out [dev]; stats->n_chunks / n_records.  Graph-capturable. */
int32_t vms_dpt_chunks(vms_dpt* d, uint32_t page_size, vms_chunk* out, int64_t cap,
                       vms_dpt_stats* stats, void* stream);
/* Snapshot (synchronises `stream`): per entry level (-1 empty), LRU stamp and
 * max_slots slot page ids [host]; res [host] (page_count + 1) entry << 8 | slot
 * or 0xFFFFFFFF.  Synchronises the device. */
int32_t vms_dpt_state(const vms_dpt* d, int32_t* level, int64_t* last_used, uint32_t* slots,
                      int32_t max_slots, uint32_t* res, void* stream);

/* ---- weighted k-means LOD pyramid (lod.py) -------------- */

/* NumPy's Philox bit-generator state (Generator(Philox(...)).bit_generator
 * .state: counter, key, buffer, buffer_pos, has_uint32, uinteger). */
typedef struct vms_philox {
  uint64_t counter[4];
  uint64_t key[2];
  uint64_t buffer[4];
  int32_t buffer_pos;
  int32_t has_uint32;
  uint32_t uinteger;
  uint32_t _pad;
} vms_philox;

typedef struct vms_lod_params {
  double weights[5];    /* AttributeWeights position, rotation, scale, opacity,
                           sh_dc (lod.py:26-41) */
  double scale_factor;  /* merge volume compensation (lod.py:22, :150) */
  int32_t max_iters;    /* Lloyd iteration cap (lod.py:23, :106) */
  int32_t k;            /* 0: one pyramid level (_page_pyramid, lod.py:157-176):
                           all-zero rows are padding, k = ceil(live / 2), the
                           clusters are merged into `out`; > 0: cluster_page
                           (lod.py:83-131) of every row with this k, the
                           cluster index per row into `assign_out`; -1:
                           merge_cluster (lod.py:134-154) of all rows into
                           the first row of `out` */
} vms_lod_params;

size_t vms_lod_workspace_bytes(uint32_t pages, uint32_t rows_in);

/* One CTA per page, `pages` pages of `rows_in` records (59 f32) at `in`
 * [dev]; rows_in <= 4096.  Pyramid mode writes each page's merged records
 * to the front of its `rows_out` rows of `out` [dev] (the rest zero), in
 * cluster order, exactly as _page_pyramid + merge_cluster (lod.py:134-176).
 * `rng` [dev] holds one NumPy Philox state per page and is advanced exactly
 * as the reference's draws advance it.  `status` [dev] per page: 0 ok,
 * 1 k-means inertia increased (InvariantViolation, lod.py:113-114), 2 level
 * overflow (lod.py:171-172).  Results are bit-identical to the reference. */
int32_t vms_lod_level(const float* in, uint32_t pages, uint32_t rows_in, float* out,
                      uint32_t rows_out, const vms_lod_params* params, vms_philox* rng,
                      int32_t* assign_out, int32_t* status, void* workspace,
                      size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* VMSPLAT_B200_H */
