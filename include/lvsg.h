/*
 * lvsg — B200-native drop-in for the reference `lvs` per-frame
 * reconstruct + render path (Quark, arXiv 2411.16680).
 *
 * C ABI: plain structs, pointers and sizes; no exceptions cross it; every
 * entry point returns an lvsg_status. Each function cites the reference
 * interface it replaces (paths relative to the reference's proj/ tree).
 *
 * Layouts (identical to the reference's Tensor<float> row-major layouts):
 *   image        [H, W, 3]              HWC fp32       (network.hpp:369-381)
 *   LDM depth    [L, Ho, Wo]            fp32, metres   (ldm.hpp:14-21)
 *   LDM density  [L, Ho, Wo]            fp32 in [0,1]
 *   LDM blend    [L, Ho, Wo, M]         fp32, post-softmax
 *   rgb          [Ho, Wo, 3]            fp32           (ldm.hpp:193-199)
 *   weights      build_params order     (network.hpp:244-317); conv
 *                [Cout,Cin,3,3], linear [in,out] (tape.hpp:700-706)
 */
#ifndef LVSG_H_
#define LVSG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error classes of the reference (tensor.hpp:15-25, io.hpp:18-31; CLI exit
 * codes main.cpp:670-693). >= 10: device / runtime failures. */
typedef enum {
  LVSG_OK = 0,
  LVSG_ERR_DIM = 1,      /* DimError: shape / contract violation            */
  LVSG_ERR_NUMERIC = 2,  /* NumericError: NaN / Inf                          */
  LVSG_ERR_IO = 3,       /* IoError                                          */
  LVSG_ERR_CUDA = 10,    /* CUDA runtime failure                             */
  LVSG_ERR_NO_DEVICE = 11,
  LVSG_ERR_NCCL = 12,
  LVSG_ERR_INTERNAL = 13
} lvsg_status;

/* StepConfig (network.hpp:38-44). `blocks` is the reference block grammar:
 * comma-separated Bp | U | Lc | A<h> | C (network.hpp:30-36). */
typedef struct {
  int64_t in_layers, layers, height, width, pyramid_level;
  const char* blocks;
} lvsg_step_config;

/* ModelConfig (network.hpp:46-59). */
typedef struct {
  const lvsg_step_config* steps;
  int64_t num_steps;
  int64_t channels, views, pyramid_levels;
  double upsample, near_depth, far_depth;
  int32_t ablate_render, ablate_attention, ablate_rays, direct_rgb;
} lvsg_model_config;

/* Camera (camera.hpp:14-41): pinhole, z-depth, texel centres at +0.5;
 * cam_from_world is a row-major 4x4. */
typedef struct {
  double fx, fy, cx, cy;
  int64_t width, height;
  double cam_from_world[16];
} lvsg_camera;

/* Frustum (camera.hpp:54-59). */
typedef struct {
  lvsg_camera camera;
  double near_depth, far_depth;
} lvsg_frustum;

/* One resolved step of plan_forward (network.hpp:62-72). */
typedef struct {
  int64_t in_layers, layers, in_height, in_width, height, width;
  int32_t doubled;
  int64_t level, feat_h, feat_w, render_h, render_w, collapse_count, num_tokens;
} lvsg_step_plan;

#define LVSG_MAX_STEPS 32
#define LVSG_MAX_LEVELS 16

/* ForwardPlan (network.hpp:74-78). */
typedef struct {
  int64_t num_levels;
  int64_t pyramid_h[LVSG_MAX_LEVELS], pyramid_w[LVSG_MAX_LEVELS];
  int64_t num_steps;
  lvsg_step_plan steps[LVSG_MAX_STEPS];
  int64_t out_height, out_width;
} lvsg_plan;

/* Optional LDM / diagnostics outputs of lvsg_forward (ForwardResult,
 * network.hpp:551-558). Any pointer may be NULL. Host pointers. */
typedef struct {
  float* depth;        /* [L,Ho,Wo]   */
  float* density;      /* [L,Ho,Wo]   */
  float* blend;        /* [L,Ho,Wo,M] */
  float* blend_logits; /* [L,H,W,M] pre-softmax, volume resolution */
  float* volume;       /* [L,H,W,C] final feature volume V         */
  float* deltas;       /* [L,H,W,M,C] the final step's update features */
  float* rgb;          /* [Ho,Wo,3] decoded-colour composite; direct_rgb
                          configs only (ForwardResult.rgb, network.hpp:596-601) */
} lvsg_ldm_out;

typedef struct lvsg_ctx lvsg_ctx;

/* ---- configuration (pure host, no device) ------------------------------ */

/* ModelConfig::validate (network.cpp:45-103). */
lvsg_status lvsg_validate_config(const lvsg_model_config* cfg, char* err, size_t err_len);
/* plan_forward (network.cpp:105-151). */
lvsg_status lvsg_plan_forward(const lvsg_model_config* cfg, int64_t image_h, int64_t image_w,
                              lvsg_plan* out, char* err, size_t err_len);
/* Parameter list of build_params (network.hpp:244-317): count, then per
 * index the shape (rank <= 4). */
lvsg_status lvsg_param_count(const lvsg_model_config* cfg, int64_t* count, int64_t* total_numel);
lvsg_status lvsg_param_shape(const lvsg_model_config* cfg, int64_t index, int32_t* rank,
                             int64_t dims[4]);
/* init_param_store<float>(cfg, seed) (network.hpp:354-362), bit-exact:
 * mt19937_64 + Box-Muller (rng.hpp:14-51). `out` holds total_numel floats,
 * tensors concatenated in build_params order. */
lvsg_status lvsg_init_param_store(const lvsg_model_config* cfg, uint64_t seed, float* out);

/* ---- context ------------------------------------------------------------ */

/* Creates a context bound to CUDA device `device`: validates cfg, owns the
 * device weights, one CUDA stream and the per-frame scratch arena. */
lvsg_status lvsg_create(const lvsg_model_config* cfg, int32_t device, lvsg_ctx** out);
void lvsg_destroy(lvsg_ctx* ctx);
/* Message of the last failure on this context (or of lvsg_create when ctx
 * is NULL). */
const char* lvsg_last_error(const lvsg_ctx* ctx);

/* bind_params(cfg, store) (network.hpp:330-339): `count` tensors in
 * build_params order with their shapes (ranks[i], dims concatenated). Shape
 * mismatches and wrong counts -> LVSG_ERR_DIM. */
lvsg_status lvsg_load_weights(lvsg_ctx* ctx, int64_t count, const float* const* tensors,
                              const int32_t* ranks, const int64_t* dims);
/* The same store as a QNTC named-tensor container (pack_tensors,
 * io.cpp:100-124): `count` f32 entries bound by position as above (names are
 * carried, not used for binding). A malformed container -> LVSG_ERR_IO with
 * unpack_tensors' message (io.cpp:126-171); an f64 entry -> LVSG_ERR_DIM
 * (NamedTensor::as_f32's SchemaError, io.cpp:86-90). */
lvsg_status lvsg_load_weights_qntc(lvsg_ctx* ctx, const void* bytes, size_t len);
/* NetParams member path of build_params tensor `index`
 * ("encoder.levels.0.res1.w1", network.hpp:95-132). */
lvsg_status lvsg_param_name(const lvsg_model_config* cfg, int64_t index, char* out, size_t len);
/* init_param_store(cfg, seed) packed as a QNTC container with those names:
 * *len receives the byte size; out == NULL only sizes it. */
lvsg_status lvsg_pack_param_store_qntc(const lvsg_model_config* cfg, uint64_t seed, void* out,
                                       size_t cap, size_t* len);
/* init_params(cfg, seed) on the host, uploaded (network.hpp:321-328). */
lvsg_status lvsg_init_weights(lvsg_ctx* ctx, uint64_t seed);

/* forward() (network.hpp:562-603) on host buffers: M images [H,W,3] (the
 * encoder resolution), M cameras, target frustum. The LDM stays resident on
 * the device for lvsg_render; `out` (optional) receives host copies. */
lvsg_status lvsg_forward(lvsg_ctx* ctx, int64_t views, const float* const* images, int64_t height,
                         int64_t width, const lvsg_camera* cams, const lvsg_frustum* target,
                         const lvsg_ldm_out* out);
/* render_target() (ldm.hpp:193-199) of the resident LDM against M images
 * [Hr,Wr,3] with their own cameras (the render resolution may differ from
 * the encoder's). rgb_out: host [Ho,Wo,3]. */
lvsg_status lvsg_render(lvsg_ctx* ctx, int64_t views, const float* const* images, int64_t height,
                        int64_t width, const lvsg_camera* cams, float* rgb_out);
/* forward() + render_target() in one call (the CLI forward-demo path,
 * main.cpp:533-541). enc_images == NULL: the resident feature pyramid of
 * lvsg_encode_device (enc_h x enc_w, complete on the context's stream,
 * lvsg_stream) is used instead of uploading and encoding. */
lvsg_status lvsg_forward_render(lvsg_ctx* ctx, int64_t views, const float* const* enc_images,
                                int64_t enc_h, int64_t enc_w, const lvsg_camera* enc_cams,
                                const float* const* render_images, int64_t render_h,
                                int64_t render_w, const lvsg_camera* render_cams,
                                const lvsg_frustum* target, float* rgb_out);

/* Pipelined host-buffer frames (video, config 4): lvsg_submit_frame enqueues
 * the work of lvsg_forward_render and returns at once with a ticket;
 * lvsg_wait_frame(ticket) blocks until that frame's rgb_out is filled and
 * reports its errors. Two frames may be in flight (submitting a third waits
 * for the oldest, and reports its errors; waiting a retired ticket returns
 * LVSG_OK at once): frame k+1's uploads run under frame k's compute and
 * frame k's read-back on its own stream. Host buffers must stay valid (and,
 * for overlap, be pinned) until the frame's wait returns.
 * lvsg_forward_render == submit + wait. */
lvsg_status lvsg_submit_frame(lvsg_ctx* ctx, int64_t views, const float* const* enc_images,
                              int64_t enc_h, int64_t enc_w, const lvsg_camera* enc_cams,
                              const float* const* render_images, int64_t render_h,
                              int64_t render_w, const lvsg_camera* render_cams,
                              const lvsg_frustum* target, float* rgb_out, int64_t* ticket);
lvsg_status lvsg_wait_frame(lvsg_ctx* ctx, int64_t ticket);

/* Input-side decimation: the caller passes only the
 * full-resolution views (e.g. 1080p); they are uploaded once, and the
 * encoder input is their resize_bilinear to (enc_h, enc_w) on the device
 * (tape.hpp:858-917, per channel of the HWC image, as the reference's
 * chw_to_hwc(resize_bilinear(hwc_to_chw(x)))) seen by cameras
 * Camera::scaled(enc_w, enc_h) (camera.cpp:67-77) of the render cameras.
 * Otherwise identical to lvsg_forward_render / lvsg_submit_frame (same
 * tickets, same two frames in flight). */
lvsg_status lvsg_forward_render_decimated(lvsg_ctx* ctx, int64_t views,
                                          const float* const* render_images, int64_t render_h,
                                          int64_t render_w, const lvsg_camera* render_cams,
                                          int64_t enc_h, int64_t enc_w,
                                          const lvsg_frustum* target, float* rgb_out);
lvsg_status lvsg_submit_frame_decimated(lvsg_ctx* ctx, int64_t views,
                                        const float* const* render_images, int64_t render_h,
                                        int64_t render_w, const lvsg_camera* render_cams,
                                        int64_t enc_h, int64_t enc_w, const lvsg_frustum* target,
                                        float* rgb_out, int64_t* ticket);
/* The decimation alone on DEVICE buffers: src [M,h,w,3] -> dst
 * [M,out_h,out_w,3] (resize_bilinear per channel), on `stream` (NULL: the
 * context's stream). */
lvsg_status lvsg_decimate_views_device(lvsg_ctx* ctx, int64_t views, const float* src, int64_t h,
                                       int64_t w, float* dst, int64_t out_h, int64_t out_w,
                                       void* stream);

/* Device-resident variant: enc_images [M,He,We,3] and render_images
 * [M,Hr,Wr,3] are contiguous DEVICE buffers, rgb_out a DEVICE buffer
 * [Ho,Wo,3]; work is enqueued on `stream` (cudaStream_t, NULL = the
 * context's stream) and the call returns without synchronising.
 * enc_images == NULL: encode_inputs' convolutions are skipped and the
 * resident feature pyramid (lvsg_encode_device, He x We) is used, so one
 * encode serves several targets of the same frame. */
lvsg_status lvsg_forward_render_device(lvsg_ctx* ctx, int64_t views, const float* enc_images,
                                       int64_t enc_h, int64_t enc_w, const lvsg_camera* enc_cams,
                                       const float* render_images, int64_t render_h,
                                       int64_t render_w, const lvsg_camera* render_cams,
                                       const lvsg_frustum* target, float* rgb_out, void* stream);

/* The same with only output rows [row0, row1) rendered into rgb_out
 * ([row1-row0, Wo, 3], device): one row band of a target split across GPUs
 * (the solve is replicated; the bands are gathered by the caller). */
lvsg_status lvsg_forward_render_rows_device(lvsg_ctx* ctx, int64_t views, const float* enc_images,
                                            int64_t enc_h, int64_t enc_w,
                                            const lvsg_camera* enc_cams, const float* render_images,
                                            int64_t render_h, int64_t render_w,
                                            const lvsg_camera* render_cams,
                                            const lvsg_frustum* target, int64_t row0, int64_t row1,
                                            float* rgb_out, void* stream);

/* encode_inputs' convolutional part (network.hpp:388-395: stem, residual
 * pairs, mean pools) of views [view0, view1) of the DEVICE images
 * [views,He,We,3] into the context's resident feature pyramid. The pyramid
 * is target-independent: one encode per frame serves every target, and a
 * view-sharded encode (each GPU its own view range) is completed by an
 * all-gather of the level buffers (lvsg_pyramid_level). Enqueued on
 * `stream` (NULL = the context's stream), no synchronisation. */
lvsg_status lvsg_encode_device(lvsg_ctx* ctx, int64_t views, const float* enc_images,
                               int64_t enc_h, int64_t enc_w, int64_t view0, int64_t view1,
                               void* stream);
/* Device pointer and extent [M, H_k, W_k, C] (fp32, view-major) of pyramid
 * level k of the context's feature pyramid buffers (allocated by the first
 * encode / export at an encoder resolution). */
lvsg_status lvsg_pyramid_level(lvsg_ctx* ctx, int64_t level, float** data, int64_t dims[4]);

/* Fused pyramid exchange across GPUs (one process per GPU): export the
 * context's pyramid level buffers for encoder input enc_h x enc_w as CUDA IPC
 * handles (handles: pyramid_levels x 64 bytes), hand every other rank's
 * handles to lvsg_pyramid_import (npeers x pyramid_levels x 64 bytes, any
 * order). From then on lvsg_encode_device's last conv of every level stores
 * each pooled value into its own and every peer's level buffer over NVLink, so
 * after a stream-ordered barrier across the ranks (e.g. a one-element NCCL
 * all-reduce) every rank holds the whole pyramid with no separate
 * all-gather. The buffers stay fixed until the context is destroyed (a new
 * encoder resolution is then a DimError). */
lvsg_status lvsg_pyramid_export(lvsg_ctx* ctx, int64_t enc_h, int64_t enc_w, uint8_t* handles);
lvsg_status lvsg_pyramid_import(lvsg_ctx* ctx, int64_t npeers, const uint8_t* handles);

/* Row-band render for output sharding across GPUs: renders
 * output rows [row0,row1) of the resident LDM into rgb_out (device,
 * [row1-row0, Wo, 3]). Bit-identical to the same rows of a full render. */
lvsg_status lvsg_render_rows_device(lvsg_ctx* ctx, int64_t views, const float* render_images,
                                    int64_t render_h, int64_t render_w,
                                    const lvsg_camera* render_cams, int64_t row0, int64_t row1,
                                    float* rgb_out, void* stream);

/* Synchronise the context stream; returns the first asynchronous error. */
lvsg_status lvsg_synchronize(lvsg_ctx* ctx);

/* Per-frame kernel-launch count of the last forward_render (for the bench's
 * gpu_launches claim) and the CUDA stream the context enqueues on. */
int64_t lvsg_last_launch_count(const lvsg_ctx* ctx);
/* Per-stage device timing: when enabled, an event closes every launch group
 * (stages: conv, gather, attention, splat, collapse, render, misc);
 * lvsg_profile_read writes "stage total_ms launches" lines accumulated since
 * the last read. Adds event records, so never enabled in a timed run. */
lvsg_status lvsg_profile_enable(lvsg_ctx* ctx, int32_t on);
lvsg_status lvsg_profile_read(lvsg_ctx* ctx, char* buf, size_t len);
void* lvsg_stream(lvsg_ctx* ctx);

/* ---- stage entry points (per-stage parity, SURVEY.md §7 hard part 2) -----
 * DEVICE pointers, run on the context stream and synchronised. */

/* geo::world_points (geometry.hpp:84-129): depth [L,H,W] -> points
 * [L,H,W,3]. Out-of-range depth -> LVSG_ERR_DIM (checked on the device). */
lvsg_status lvsg_stage_world_points(lvsg_ctx* ctx, const lvsg_frustum* fr, const float* depth,
                                    int64_t L, int64_t H, int64_t W, float* points);
/* geo::footprint + CamPod::to_cam over points [P,3] (geometry.hpp:34-79,
 * :152-160): x0,x1,y0,y1 (int32, 4 per point), valid (uint8), fx,fy (f64). */
lvsg_status lvsg_stage_footprints(lvsg_ctx* ctx, const lvsg_camera* cam, const float* points,
                                  int64_t P, int32_t* taps, uint8_t* valid, double* fracs);
/* geo::gather_backproject (geometry.hpp:138-224): image [Hi,Wi,C], points
 * [P,3] -> values [P,C] (zero where invalid) and mask [P]. */
lvsg_status lvsg_stage_gather(lvsg_ctx* ctx, const lvsg_camera* cam, const float* image,
                              int64_t Hi, int64_t Wi, int64_t C, const float* points, int64_t P,
                              float* values, float* mask);
/* attend_residual (attention.hpp:248-252) in place on V [P, C] (device),
 * Δ in the reference layout [P, M, C] (backproject_stack, network.hpp:421-436),
 * wq heads x [C, C] contiguous, wo [heads*C, C], gain [C] (all device). */
lvsg_status lvsg_stage_attend(lvsg_ctx* ctx, float* V, const float* deltas, int64_t P, int64_t M,
                              int64_t heads, const float* wq, const float* wo, const float* gain,
                              int32_t zero_scores);
/* upsample_activate + render_target (ldm.hpp:249-271, :193-199) of a given
 * final volume: V [L,H,W,C], blend logits [L,H,W,M], heads w_depth / w_sigma
 * [C], images [M,Hr,Wr,3] (all device) seen through cams -> rgb [Ho,Wo,3]
 * (device). A depth outside the frustum -> LVSG_ERR_DIM (world_points). */
lvsg_status lvsg_stage_upsample_render(lvsg_ctx* ctx, const lvsg_frustum* target, const float* V,
                                       const float* logits, int64_t L, int64_t H, int64_t W,
                                       int64_t M, const float* w_depth, const float* w_sigma,
                                       const float* images, int64_t Hr, int64_t Wr,
                                       const lvsg_camera* cams, int64_t Ho, int64_t Wo,
                                       float* rgb);
/* render_to_input_view (ldm.hpp:223-244; splat geometry.hpp:230-326) of
 * V [L,H,W,C] (device) in the frustum `target` into one camera:
 * out [cam.height, cam.width, Ca+1] (device; composited appearance + alpha). */
lvsg_status lvsg_stage_render_to_view(lvsg_ctx* ctx, const lvsg_frustum* target, const float* V,
                                      int64_t L, int64_t H, int64_t W, const float* w_appear,
                                      int64_t Ca, const float* w_sigma, const float* w_depth,
                                      const lvsg_camera* cam, float* out);

/* ---- synthetic inputs (host; the benchmarks' generator) -----------------
 * RigSpec::cameras / ::target (scenes.cpp:40-60): rows*cols cameras, row
 * major; target may be NULL. */
lvsg_status lvsg_rig_cameras(int64_t rows, int64_t cols, double baseline, int64_t width,
                             int64_t height, double focal, lvsg_camera* cams,
                             lvsg_camera* target);
/* make_scene(seed, planes, scene_fr) + oracle_render per camera, f64 -> f32
 * (scenes.cpp:62-171). images: views contiguous [H_m, W_m, 3] blocks. */
lvsg_status lvsg_scene_images(uint64_t seed, int64_t planes, const lvsg_frustum* scene_fr,
                              int64_t views, const lvsg_camera* cams, float* images, char* err,
                              size_t err_len);
/* The same with every plane except the last (the backdrop wall) shifted by
 * shift_x metres along x: config 4's moving content. */
lvsg_status lvsg_scene_images_shifted(uint64_t seed, int64_t planes, const lvsg_frustum* scene_fr,
                                      double shift_x, int64_t views, const lvsg_camera* cams,
                                      float* images, char* err, size_t err_len);

/* conv3x3 (kernels_ref.hpp:72-96) on DEVICE channel-last tensors x
 * [B,H,W,Cin] -> y [B,H,W,Cout], w [Cout,Cin,3,3], b [Cout] (nullable).
 * impl: 0 auto, 1 fp32 SIMT, 2 tcgen05 3xTF32 (when Cin = Cout = 32). */
lvsg_status lvsg_stage_conv3x3(lvsg_ctx* ctx, const float* x, const float* w, const float* b,
                               float* y, int64_t B, int64_t Cin, int64_t Cout, int64_t H,
                               int64_t W, int32_t impl);
/* The fused forms used inside the solve: x with pixel stride x_pstride;
 * weights sliced to input channels [w_ci0, w_ci0+Cin) of a [Cout,w_cin,3,3]
 * tensor; optional rms_norm(x)*norm_gain on the input (conv_mlp_residual,
 * attention.hpp:262-266), GELU, and y = resid + conv (resid may alias y). */
lvsg_status lvsg_stage_conv3x3_fused(lvsg_ctx* ctx, const float* x, int64_t x_pstride,
                                     const float* w, int64_t w_cin, int64_t w_ci0, const float* b,
                                     const float* norm_gain, int32_t gelu, const float* resid,
                                     float* y, int64_t B, int64_t Cin, int64_t Cout, int64_t H,
                                     int64_t W, int32_t impl);

#ifdef __cplusplus
}
#endif

#endif /* LVSG_H_ */
