/*
 * lvs_oracle — CPU restatement (plain C11 + pthreads) of the reference's
 * per-frame path: lvs::forward (network.hpp:562-603) + lvs::render_target
 * (ldm.hpp:193-199), T = float.
 *
 * TEST INFRASTRUCTURE ONLY. It is the checker for the CUDA path (tests/,
 * __graft_entry__.smoke(), bench.py's cpu_baseline leg); the product library
 * never links or calls it.
 *
 * Parity pinned: every function restates the reference's floating-point
 * evaluation order (kernels_ref.hpp:5-11, no FP contraction) so results are
 * BIT-IDENTICAL to the reference built from /root/reference (oracle/_ref),
 * checked by tests/test_oracle.py against that build and against the FNV-1a
 * golden hash the survey recorded for config 1.
 * Threads only split independent outputs; per-output order is fixed, so the
 * thread count never changes a bit.
 */
#ifndef LVS_ORACLE_H_
#define LVS_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "../include/lvsg.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Thread count for all oracle calls (default: LVSO_THREADS env or 1). */
void lvso_set_threads(int n);

/* forward<float> + render_target<float>. Images contiguous [M,H,W,3];
 * weights flat in build_params order (network.hpp:244-317). Any output may be
 * NULL; render is skipped when render_images is NULL. Returns 0 or an
 * lvsg_status class (1 = DimError). */
int lvso_forward_render(const lvsg_model_config* cfg, int64_t M, const float* enc_images,
                        int64_t He, int64_t We, const lvsg_camera* enc_cams,
                        const float* render_images, int64_t Hr, int64_t Wr,
                        const lvsg_camera* render_cams, const lvsg_frustum* target,
                        const float* weights, float* rgb, float* depth, float* density,
                        float* blend, float* blend_logits, float* volume, char* err,
                        size_t errlen);
/* The same with ForwardResult's two remaining fields: deltas [L,H,W,M,C]
 * (the final step's update features) and, under direct_rgb, rgb [Ho,Wo,3]
 * (ForwardResult.rgb, network.hpp:596-601). Either may be NULL. */
int lvso_forward_render_ex(const lvsg_model_config* cfg, int64_t M, const float* enc_images,
                           int64_t He, int64_t We, const lvsg_camera* enc_cams,
                           const float* render_images, int64_t Hr, int64_t Wr,
                           const lvsg_camera* render_cams, const lvsg_frustum* target,
                           const float* weights, float* rgb, float* depth, float* density,
                           float* blend, float* blend_logits, float* volume, float* deltas,
                           float* rgb_direct, char* err, size_t errlen);

/* Stage restatements for per-stage parity. */
int lvso_world_points(const lvsg_frustum* fr, const float* depth, int64_t L, int64_t H, int64_t W,
                      float* points);
void lvso_footprints(const lvsg_camera* cam, const float* points, int64_t P, int32_t* taps,
                     uint8_t* valid, double* fracs);
void lvso_gather(const lvsg_camera* cam, const float* image, int64_t Hi, int64_t Wi, int64_t C,
                 const float* points, int64_t P, float* values, float* mask);
void lvso_upsample_activate(const lvsg_frustum* fr, const float* V, int64_t L, int64_t H, int64_t W,
                            int64_t C, const float* w_depth, const float* w_sigma,
                            const float* logits, int64_t M, int64_t Ho, int64_t Wo, float* depth,
                            float* density, float* blend);
int lvso_render_target(const lvsg_frustum* fr, const float* depth, const float* density,
                       const float* blend, int64_t L, int64_t Ho, int64_t Wo, int64_t M,
                       const float* images, int64_t Hr, int64_t Wr, const lvsg_camera* cams,
                       float* rgb);
/* attend_residual (attention.hpp:248-252): V [P,C] in place, deltas [P,M,C],
 * wq heads x [C,C] contiguous, wo [heads*C,C], gain [C]. */
void lvso_attend_residual(float* V, const float* D, int64_t P, int64_t C, int64_t M,
                          int64_t heads, const float* wq, const float* wo, const float* gain,
                          int zero);
/* render_to_input_view (ldm.hpp:223-244) -> out [cam.height, cam.width, Ca+1];
 * returns nonzero when world_points saw an out-of-frustum depth. */
int lvso_render_to_view(const lvsg_frustum* fr, const float* V, int64_t L, int64_t H, int64_t W,
                        int64_t C, int64_t Ca, const float* w_appear, const float* w_sigma,
                        const float* w_depth, const lvsg_camera* cam, float* out);
/* Validity-margin trace of the forward's gathers and splats (parity
 * attribution): rows of 8 floats (step, kind 0 gather / 1 splat, view,
 * layer, y, x, signed margin px, u-or-v) for every footprint within tol px of
 * its validity boundary; buf NULL disables. Not thread-safe across calls. */
void lvso_trace_margins(double tol, float* buf, int64_t cap);
int64_t lvso_trace_count(void);
/* conv3x3 (kernels_ref.hpp:72-96), CHW / OIHW, zero pad by tap skipping. */
void lvso_conv3x3(const float* x, const float* w, const float* b, float* y, int64_t Cin,
                  int64_t Cout, int64_t H, int64_t W);

#ifdef __cplusplus
}
#endif

#endif
