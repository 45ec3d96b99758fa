// Launchers for the lvsg device kernels. All tensors are fp32, channel-last
// (HWC) unless stated; all launches are asynchronous on `st`.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace lvsg {

// Programmatic dependent launch. Every kernel of the path opens with
// pdl_grid_sync() (allow the next kernel to launch, then wait until the
// previous one has completed and its memory is visible), so it is correct to
// launch any of them with the attribute. It is set only for the persistent
// tensor-core kernels (conv3x3_tc, attention: one CTA per SM, > 200 KB smem):
// their CTAs cannot co-reside with each other, so an early launch only
// overlaps the predecessor's tail with their prologue, whereas small
// dependents launched early would sit in griddepcontrol.wait beside a
// running persistent kernel and slow it down (measured: 111.6 vs 107.4
// frames/s). LVSG_PDL=0 turns the attribute off everywhere.
bool pdl_enabled();
bool pdl_all();  // LVSG_PDL=2: the attribute on every launch (measurement switch)

__device__ __forceinline__ void pdl_grid_sync() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Opts `kernel` into `bytes` of dynamic shared memory on the CURRENT device,
// once per (device, kernel); thread-safe (a process may drive several GPUs
// and several contexts from several threads).
void smem_optin(const void* kernel, int bytes);
// Multiprocessor count of the current device (cached per device).
int sm_count();

template <typename... KArgs, typename... Args>
inline void launch_pdl(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = ((pdl || pdl_all()) && pdl_enabled()) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t st, Args... args) {
  launch_pdl(false, kernel, grid, block, smem, st, args...);
}

// ---- conv3x3 (kernels_ref.hpp:72-96 semantics, zero padding) -------------
// Input = channel concatenation of up to 3 sources, each [B, H, W, C_i] with
// pixel stride `pstride` floats and batch stride `bstride` floats. Optional
// per-pixel rms-norm transform on the input (x * rinv[b,pix]) * gain[c]
// (fusing conv_mlp_residual's rms_norm, attention.hpp:262-266). Epilogue:
// + bias, optional GELU, optional residual (out = resid + y; may alias out).
struct ConvSrc {
  const float* ptr;
  int C;
  int pstride;
  long long bstride;
};
struct ConvArgs {
  ConvSrc src[3];
  int nsrc;
  int Cin, Cout, H, W, B;
  const float* w;     // [Cout, Cin, 3, 3]
  const float* bias;  // [Cout] or null
  const float* rinv;  // [B, H, W] or null
  const float* gain;  // [Cin] (with rinv)
  int gelu;
  float* out;
  int out_pstride;
  long long out_bstride;
  const float* resid;  // or null
  int res_pstride;
  long long res_bstride;
  // input-channel slice of the weight tensor: w is [Cout, w_cin, 3, 3] and
  // this conv uses channels [w_ci0, w_ci0 + Cin) (0 = w_cin = Cin when unset)
  int w_cin, w_ci0;
  // tensor-core weight image (conv3x3_tc_prepare) for conv3x3_tc; required there
  const void* wsplit;
  int w_early;  // the image is settled: bulk-load it before griddepcontrol.wait
  // launch conv3x3_tc with programmatic dependent launch (its prologue overlaps
  // the previous kernel's tail); only when nothing it reads before its grid
  // dependency wait was produced by that kernel
  int pdl;
  // conv3x3_tc only: one extra single-channel input folded into the epilogue
  // (the feedback's alpha channel of the update-CNN stem): out += sum_tap
  // alpha(y+dy-1, x+dx-1) * w[co][alpha_ci][tap], alpha at alpha[b*alpha_bstride
  // + pix*alpha_pstride] (a separate kernel instantiation)
  const float* alpha;
  int alpha_pstride, alpha_ci;
  long long alpha_bstride;
  // conv3x3_tc only: also write the 2x2 mean pool of the output (the encoder's
  // mean_pool2, same summation order) to pool_out [B, H/2, W/2, 32]
  float* pool_out;
  long long pool_bstride;
  // ... and the same pooled values stored into up to 7 peer GPUs' copies of
  // the pyramid level (same offsets, mapped over NVLink by CUDA IPC): the
  // view-sharded encode's exchange fused into the producing epilogue
  float* pool_peer[7];
  int npool_peer;
  // Cin = 3 stem only: host copy of the weights [32][3][3][3] and bias [32]
  // (the encoder stem, bound at weight load). The stem kernel then takes
  // them by value in its parameter space, so every FMA reads its weight as
  // a constant-bank operand (no shared-memory weight loads).
  const float* stem_host;
  // tcgen05 conv only: set bit 2 (atomicOr) when an operand of the fp16
  // split overflows (|x| >= 65520 rounds to inf in the hi term): the split
  // would be silently wrong, so the call reports LVSG_ERR_NUMERIC instead
  int* ovf;
  // debug builds with LVSG_TIMELINE: 1-based slot of this launch in the conv
  // timeline (globaltimer at entry / after the grid dependency wait / exit)
  int tl_slot;
};
// LVSG_TIMELINE builds: reset / read the conv timeline ([slot][4]: entry,
// ready, exit, CTAs); other builds: no-op / -1
void conv_timeline_reset();
int conv_timeline_read(unsigned long long* out, int slots);
__host__ __device__ inline int w_cin_of(const ConvArgs& a) { return a.w_cin ? a.w_cin : a.Cin; }
// Dispatches to the tcgen05 3xTF32 kernel when it applies (Cin = Cout = 32,
// one 16-byte-aligned source), else to the fp32 SIMT kernel. impl: 0 auto,
// 1 SIMT, 2 tcgen05 (unsupported shapes fall back to SIMT).
void conv3x3(const ConvArgs& a, cudaStream_t st, int impl = 0);
void conv3x3_simt(const ConvArgs& a, cudaStream_t st);
bool conv3x3_uses_tc(const ConvArgs& a, int impl = 0);
bool conv3x3_tc_supported(const ConvArgs& a);
void conv3x3_tc(const ConvArgs& a, cudaStream_t st);
// Bytes of one tensor-core weight image: the [tap][8-channel plane][64 rows]
// fp16 hi / lo' split of w[:, w_ci0 : w_ci0 + 32] in the kernel's shared
// memory layout, loaded by one bulk copy per CTA.
constexpr size_t kConvTcWeightBytes = 9 * 4 * 64 * 16;
void conv3x3_tc_prepare(const ConvArgs& a, void* dst, cudaStream_t st);
// Which conv runs: 1 SIMT / stem, 2 tensor core (impl: 0 auto = tensor core
// where supported; LVSG_CONV=simt forces the SIMT kernel).
int conv3x3_path(const ConvArgs& a, int impl = 0);

// ---- elementwise / layout ------------------------------------------------
void fill_rows(float* out, const float* row, int64_t rows, int C, cudaStream_t st);
void fill_layers(float* out, const float* per_layer, int L, int64_t P, cudaStream_t st);
// depth[l, :] = T(1 / (double(T((l+0.5)/L)) * inv_span + inv_far)) (network.hpp:469-475)
void fill_anchor_depths(float* out, int L, int64_t P, double inv_span, double inv_far,
                        cudaStream_t st);
void mean_pool2(const float* in, float* out, int B, int H, int W, int C, cudaStream_t st);
// resize_bilinear of [B,H,W,C] (tape.hpp:858-917, per channel).
void resize_hwc(const float* in, float* out, int B, int H, int W, int C, int Ho, int Wo,
                cudaStream_t st);
// rms_norm reciprocal per row: rinv = 1/sqrt(mean(x^2)+1e-6) (tape.hpp:779-785).
void rms_rinv(const float* x, float* rinv, int64_t rows, int C, cudaStream_t st);

// ---- encoder ray encodings (geometry.hpp:343-391, network.hpp:397-413) -----
struct RayBaseCam {
  double Rwc_in[9];  // grid camera R^T
  double o[3];       // input centre in the target frame
  double fx, fy, cx, cy;  // grid camera intrinsics
};
struct RayBaseArgs {
  double Rcw_t[9];
  double tfx, tfy, inv_span, half_w, half_h;
  int h, w, M;
};
void ray_base(const RayBaseCam* cams_dev, const RayBaseArgs& a, float* base, cudaStream_t st);
// rays_k = resize(base -> Hk,Wk) @ ray_proj [32,C]
// proj_host (optional): host copy of proj ([32, C], C = 32) for the
// parameter-space kernel.
void ray_project(const float* base, int M, int hK, int wK, int Hk, int Wk, const float* proj,
                 int C, float* out, cudaStream_t st, const float* proj_host = nullptr);

// ---- geometry --------------------------------------------------------------
// Δ[p, m, :] = gather of feats[m] ([M, Hf, Wf, C]) at world_point(p) through
// cams[m] (backproject_stack, network.hpp:421-436; invalid -> 0), stored
// texel-major per view: deltas[m][p][C] (one contiguous C-float row per
// texel-view; Stage 2 reads 128-texel slices of it with 2-D TMA boxes).
void gather_stack(const float* feats, int M, int Hf, int Wf, int C, const DevCam* cams_dev,
                  const DevRayCam& rc, const float* depth, int L, int H, int W, float* deltas,
                  cudaStream_t st);

// Per-pixel strides of the render-to-input-view buffers, padded to 16 bytes
// so every row moves as float4 / vector atomics and feeds TMA: the payload
// and the composited feedback carry K = Ca+1 channels, the splat
// accumulators K+1 (the bilinear weight sum).
__host__ __device__ inline int pay_stride(int K) { return (K + 3) & ~3; }
// Row stride of the splat's input payload [P, K]: 32-byte rows, so the
// reduction loads each row with 256-bit loads (C = 32: 40 floats).
__host__ __device__ inline int payload_stride(int K) { return (K + 7) & ~7; }
__host__ __device__ inline int acc_stride(int K) { return (K + 1 + 3) & ~3; }

// render_to_input_view decode (ldm.hpp:229-235): payload [P, Ca+1] =
// [sigmoid(V w_a), sigmoid(V w_sigma)], depth [P] = activate(V w_depth) and
// world points [P,3].
// w_host (optional, C = Ca = 32): host copy of the three heads as [k][36]
// (appear | sigma | depth | 0 0) for the parameter-space kernel.
void decode_payload(const float* V, int L, int H, int W, int C, const float* w_appear, int Ca,
                    const float* w_sigma, const float* w_depth, const DepthAct& da,
                    const DevRayCam& rc, float* payload, float* depth, float* points,
                    cudaStream_t st, const float* w_host = nullptr);
// splat_accumulate (geometry.hpp:230-264) + normalise + composite
// (splat_det.cu): every view pixel sums its taps in the reference's order
// (bit-identical from run to run). scratch holds
// splat_det_scratch_ints(L*PL*M, M*L*Hv*Wv) ints.
size_t splat_det_scratch_ints(int64_t pairs, int64_t bins);
void splat_det(const float* payload, const float* points, int L, int PL, int K,
               const DevCam* cams_dev, int M, int Hv, int Wv, int* scratch, float* out,
               cudaStream_t st);

// ---- attention / fusion ----------------------------------------------------
// Δ from the reference layout [P, M, C] (network.hpp:421-436) into the
// kernels' layout [M][P][C] (texel-major per view; stage entry points).
void deltas_to_view_major(const float* src, float* dst, int64_t P, int M, int C, cudaStream_t st);
// Stream-ordered copy of `bytes` from pinned (device-mapped) host memory by a
// kernel rather than a copy engine: a small per-frame table then never queues
// behind a bulk image upload on another stream.
void copy_from_pinned(void* dst, const void* pinned_src, size_t bytes, cudaStream_t st);
// V += OTM(rms_norm(V), Δ) (attention.hpp:207-252), in place. scratch:
// attend_scratch_floats(P, C, M, heads) floats of device memory from the
// caller's arena (the generic fallback's per-texel rows; none for the
// tensor-core kernel).
// wimg (optional): attend_tc_prepare's image of (wq, wo), 16-byte aligned.
// ovf (optional): bit 2 set when an fp16-split operand overflows (ConvArgs.ovf).
void attend(float* V, const float* deltas, int64_t P, int C, int M, int heads, const float* wq,
            const float* const* wq_heads, const float* wo, const float* gain, int zero_scores,
            float* scratch, const void* wimg, bool wimg_early, int* ovf, cudaStream_t st);
size_t attend_scratch_floats(int64_t P, int C, int M, int heads);
// tcgen05 fused attention (attn_tc.cu): C = 32, h in {1,2,4},
// M in {2,4,8,16}; returns false otherwise.
bool attend_tc_supported(int C, int M, int heads);
bool attend_tc(float* V, const float* deltas, int64_t P, int C, int M, int heads, const float* wq,
               const float* wo, const float* gain, int zero_scores, const void* wimg,
               bool wimg_early, int* ovf, cudaStream_t st);
// The tensor-core attention's pre-split weight image (bytes; 0: no kernel
// for this head count) and the kernel that makes it.
size_t attend_tc_weight_bytes(int heads);
void attend_tc_prepare(const float* wq, const float* wo, int heads, void* dst, int* ovf,
                       cudaStream_t st);
// logits [P, M] = <rms_norm(V,g) W_blend, Δ_m> / sqrt(C) (network.hpp:539-549).
void blend_logits(const float* V, const float* deltas, int64_t P, int C, int M,
                  const float* blend_w, const float* gain, float* logits, cudaStream_t st,
                  const float* blend_w_host = nullptr);
// layer_collapse (network.hpp:440-455): V [L,H,W,C] -> out [L/2,H,W,C].
void layer_collapse(const float* V, int L, int64_t PL, int C, const float* w1, const float* b1,
                    const float* w2, const float* b2, float* out, cudaStream_t st);
// layer_collapse on tcgen05 (collapse_tc.cu, C = 32): wimg is
// collapse_tc_prepare's split image of (w1, w2), made once per binding;
// false when the shape does not apply.
size_t collapse_tc_weight_bytes();
void collapse_tc_prepare(const float* w1, const float* w2, void* dst, int* ovf, cudaStream_t st);
bool layer_collapse_tc(const float* V, int L, int64_t PL, int C, const float* wimg,
                       const float* b1, const float* b2, float* out, int* ovf, cudaStream_t st);
// rays_k = resize(base) @ ray_proj on tcgen05 (collapse_tc.cu, C = 32);
// wimg: ray_tc_prepare's split image of ray_proj [32, 32].
size_t ray_tc_weight_bytes();
void ray_tc_prepare(const float* proj, void* dst, int* ovf, cudaStream_t st);
bool ray_project_tc(const float* base, int M, int hK, int wK, int Hk, int Wk, const float* wimg,
                    float* out, int* ovf, cudaStream_t st);
// C = 32 specialisations (fast32.cu); return false when the shape differs.
bool layer_collapse32(const float* V, int L, int64_t PL, int C, const float* w1, const float* b1,
                      const float* w2, const float* b2, float* out, cudaStream_t st);
bool blend_logits32(const float* V, const float* deltas, int64_t P, int C, int M,
                    const float* blend_w, const float* gain, float* logits, cudaStream_t st,
                    const float* blend_w_host = nullptr);
bool decode_payload32(const float* V, int L, int H, int W, int C, const float* w_appear, int Ca,
                      const float* w_sigma, const float* w_depth, const DepthAct& act,
                      const DevRayCam& rc, float* payload, float* depth, float* points,
                      cudaStream_t st, const float* w_host = nullptr);
// out[p] = V[p,:] . w (decode_linear with K = 1), optionally activated depth.
// Both pre-activation heads (out_a = V w_a, out_b = V w_b) in one pass over V.
void decode_scalar2(const float* V, int64_t P, int C, const float* wa, float* outa, const float* wb,
                    float* outb, cudaStream_t st);
void decode_scalar(const float* V, int64_t P, int C, const float* w, float* out, int L,
                   int64_t PL, const DepthAct* act, cudaStream_t st);

// ---- Stage 3 + 4 ------------------------------------------------------------
constexpr int kRenderParamViews = 32;
struct RenderArgs {
  const float* pre_d;   // [L,H,W]
  const float* pre_s;   // [L,H,W]
  const float* logits;  // [L,H,W,M]
  int L, H, W, M, Ho, Wo;
  int row0, row1;  // output rows rendered (row band)
  DepthAct act;
  DevRayCam rc;           // target camera re-digitised to (Wo, Ho)
  const DevCam* cams;     // [M] render cameras (device)
  DevCam pc[kRenderParamViews];  // the same by value (M <= 32; the view-count kernels)
  FastCam fc[kRenderParamViews];  // ... folded for the fast footprint (fast_cam)
  int pc_valid;                  // pc holds the M cameras
  const float* images;    // [M, Hr, Wr, 3]
  int Hr, Wr;
  float* rgb;             // [row1-row0, Wo, 3]
  float near_depth, far_depth;
  int* bad_depth;         // set when a depth leaves [near-slack, far+slack]
  double slack_lo, slack_hi;
};
// The render's folded camera (FastCam, common.cuh) of a DevCam, on the host.
FastCam fast_cam(const DevCam& d);
// upsample_activate + render_target fused (ldm.hpp:193-199, :249-271).
void render_fused(const RenderArgs& a, cudaStream_t st);
// ForwardResult.rgb of a direct_rgb config (network.hpp:596-601): pre_a =
// decode_linear(V, w_appear) [L,H,W,3] -> out [Ho,Wo,3].
void direct_rgb(const RenderArgs& a, const float* pre_a, float* out, cudaStream_t st);
// decode_linear (ldm.hpp:58-67): out[p, j] = sum_k V[p, k] w[k, j], k ascending.
void decode_linear(const float* V, int64_t P, int C, const float* w, int K, float* out,
                   cudaStream_t st);
// upsample_activate only (materialised LDM for lvsg_forward outputs).
void upsample_activate(const RenderArgs& a, float* depth, float* density, float* blend,
                       cudaStream_t st);

// ---- stage entry points (per-stage parity) ----------------------------------
void stage_world_points(const DevRayCam& rc, const float* depth, int L, int H, int W,
                        float* points, double lo, double hi, int* bad, cudaStream_t st);
void stage_footprints(const DevCam& cam, const float* points, int64_t P, int32_t* taps,
                      uint8_t* valid, double* fracs, cudaStream_t st);
void stage_gather(const DevCam& cam, const float* image, int Hi, int Wi, int C,
                  const float* points, int64_t P, float* values, float* mask, cudaStream_t st);

}  // namespace lvsg
