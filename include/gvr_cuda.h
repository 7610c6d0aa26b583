/* gvr_cuda.h — C ABI of the B200-native VoGE render path (sm_100a).
 *
 * Drop-in boundary for the reference's C++ render API
 * (namespace gvr, static library `gvr`, /root/reference/proj):
 *
 *   reference (proj/include/gvr/...)                           replaced by
 *   ----------------------------------------------------------  -----------------------------
 *   GaussianScene::validate            types.hpp:41, types.cpp:31  gvr_scene_set (validates once
 *                                                                   per upload, on the device)
 *   Camera::validate / SelectionConfig::validate
 *                                      types.cpp:44, tracer.cpp:8   gvr_render (host checks,
 *                                                                   same messages)
 *   RenderBuffers render(scene, camera, cfg, threads)
 *                                      blender.hpp:40-41            gvr_render(tape = context tape)
 *   ForwardResult render_with_tape(scene, camera, cfg, threads)
 *                                      grad.hpp:41-42               gvr_render(tape)
 *   detail::render_core(..., traced_out, cam_scene_out)
 *                                      blender.hpp:53-56            gvr_render + gvr_tape_traced +
 *                                                                   gvr_tape_cam_scene
 *   PixelKernelMap::dropped_behind_camera
 *                                      tracer.hpp:39                gvr_tape_dropped_behind_camera
 *   RenderBuffers::weight_store        blender.hpp:24               gvr_render_outputs.topk_idx/topk_w
 *   GradientBundle backward(tape, d_image, d_alpha, flags)
 *                                      grad.hpp:53-54               gvr_backward
 *   double ScalarLoss::value(buf, d_image*, d_alpha*)
 *                                      grad.hpp:68, grad.cpp:201    gvr_scalar_loss
 *   SampledAttributes sample_attributes(observed, scene, camera, cfg, normalized, threads)
 *                                      sampler.hpp:23-25            gvr_sample_attributes
 *   RenderBuffers resynthesize(attrs, scene, camera, cfg, threads)
 *                                      sampler.hpp:29-30            gvr_scene_resynthesize + gvr_render
 *   double transmittance_at(traced, tau, t)
 *                                      blender.hpp:29               gvr_tape_transmittance (per pixel)
 *   normalized_weights(RayBlend, eps)  blender.hpp:36               gvr_tape_normalized_weights
 *   Image shade_lambert(normals, alpha, depth, camera, light_pos, light_color)
 *                                      blender.hpp:46-47            gvr_shade_lambert
 *   ShapeRegularizer::make / edge_reg / laplacian_reg
 *                                      fit.hpp:50-67                gvr_regularizer_create / gvr_edge_reg /
 *                                                                   gvr_laplacian_reg
 *   ValidationError (std::runtime_error)
 *                                      types.hpp:19-22              return GVR_ERR_VALIDATION +
 *                                                                   gvr_last_error() (same text)
 *
 * Conventions (identical to the reference):
 *   centers[K*3]; inv_cov[K*9] = Sigma^-1 row-major; attr[K*D]; FP64.
 *   camera: rotation row-major, x_cam = R x_obj + T; pixel (i, j) = (row, col),
 *   pixel centres at integers, i pairs with oy; images H*W*C, channels interleaved,
 *   C = max(D, 1) for the image (zero channel when D == 0), 1 for alpha and depth.
 *   Per-pixel lists ascending by (l, kernel index), padded to k_prime with -1.
 *
 * Memory: every pointer argument may be HOST memory (pageable or pinned) or
 * DEVICE memory of the context's device; the library detects which with
 * cudaPointerGetAttributes and copies on the context's stream. All work is
 * enqueued on the context stream; calls that return host data synchronise.
 *
 * Errors: 0 = ok, 1 = validation (the reference throws gvr::ValidationError),
 * 2 = runtime / CUDA. The message is returned by gvr_last_error(ctx).
 * There is no CPU fallback: without a usable sm_100 device every call fails
 * with GVR_ERR_RUNTIME.
 */
#ifndef GVR_CUDA_H
#define GVR_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GVR_OK 0
#define GVR_ERR_VALIDATION 1
#define GVR_ERR_RUNTIME 2

typedef struct gvr_context gvr_context;
typedef struct gvr_scene gvr_scene;
typedef struct gvr_tape gvr_tape;
typedef struct gvr_graph gvr_graph;
typedef struct gvr_regularizer gvr_regularizer;

/* gvr::Camera (types.hpp:46-56) */
typedef struct {
    double rotation[9]; /* row-major */
    double translation[3];
    double focal, ox, oy;
    int32_t height, width;
} gvr_camera;

/* gvr::SelectionConfig (tracer.hpp:18-25); defaults eta 0.01, k_prime 20, coarse on, 8 */
typedef struct {
    double eta;
    int32_t k_prime;
    int32_t coarse_enabled;
    int32_t coarse_downsample;
} gvr_selection;

/* gvr::GradFlags (grad.hpp:46-49) */
typedef struct {
    int32_t through_transmittance;
    int32_t through_density;
} gvr_grad_flags;

/* Outputs of a render; every field nullable (host or device pointers). */
typedef struct {
    double* image;    /* H*W*max(D,1) */
    double* alpha;    /* H*W */
    double* depth;    /* H*W */
    int32_t* topk_idx; /* H*W*k_prime, -1 padded        (weight_store indices) */
    double* topk_w;    /* H*W*k_prime, 0 padded         (weight_store weights) */
} gvr_render_outputs;

/* gvr::GradientBundle (grad.hpp:13-22); every field nullable (host or device). */
typedef struct {
    double* d_center;      /* K*3 */
    double* d_inv_cov;     /* K*9 row-major, exactly symmetric */
    double* d_attr;        /* K*D */
    double* d_rotation;    /* 9 row-major */
    double* d_translation; /* 3 */
} gvr_gradients;

/* SHA-256 prefix of the sources the library was built from (build.py:
 * source_hash); the Python loader refuses a library that does not match. */
const char* gvr_build_hash(void);

/* ---- context: device, stream, scratch arenas ---------------------------- */
int gvr_context_create(int device, gvr_context** out);
void gvr_context_destroy(gvr_context* ctx);
const char* gvr_last_error(const gvr_context* ctx);
/* Asynchronous host buffers (on != 0): gvr_scene_set, gvr_render, gvr_scalar_loss
 * and gvr_backward with HOST pointers enqueue their copies and return without
 * synchronising (host buffers should be pinned). Inputs are copied on the context
 * stream; device->host copies of a call's outputs drain on a second stream of the
 * context while the context stream runs the next call (the next call of the same
 * kind on the tape waits for them). Results are valid after gvr_context_synchronize
 * (both streams); the checks that need the host then are deferred: scene
 * validation -> gvr_scene_check, non-finite outputs -> gvr_tape_check_finite. Lets
 * a caller pipeline steps over several contexts (one step's copies under the
 * others' kernels). Synchronises when switched. */
int gvr_context_set_async(gvr_context* ctx, int on);
/* Use an external cudaStream_t (NULL = the context's own stream). */
int gvr_context_set_stream(gvr_context* ctx, void* cuda_stream);
void* gvr_context_stream(gvr_context* ctx);
int gvr_context_synchronize(gvr_context* ctx);
/* Instrumentation: kernels of this library launched since creation; calls into
 * device-wide libraries (none on the render path: always 0). */
int64_t gvr_context_launch_count(const gvr_context* ctx);
int64_t gvr_context_library_call_count(const gvr_context* ctx);
/* Per-stage device time via CUDA events around each launch (off by default).
 * Stages: 0 project + bin count, 1 bin emit, 2 tile order + list layout,
 * 3 select, 4 blend, 5 loss, 6 backward pixels, 7 record layout + records +
 * finish (object space). Enabling resets the accumulators. */
int gvr_context_enable_timing(gvr_context* ctx, int on);
int gvr_context_stage_times(gvr_context* ctx, double* ms, int64_t* count, int n);
/* Calibration for the roofline: FMA-chain peak of the FP32 (kind 0) or FP64
 * (kind 1) pipe on this device, FLOP/s (FMA = 2). */
int gvr_measure_pipe_peak(gvr_context* ctx, int kind, double* flops);
/* Test hook: FP32 pre-filter guard band on q (default 0.02); a huge value sends
 * every candidate through the exact FP64 trace. Results must not change. */
int gvr_context_set_prefilter_guard(gvr_context* ctx, double guard);
/* Verification mode: the blend evaluates every pair term from the exact FP64
 * trace and erfc (the reference's arithmetic, ~1e-15) instead of the FP32
 * closed-form pipeline. Slow; used by gradcheck's finite differences. */
int gvr_context_set_precise(gvr_context* ctx, int on);
/* Camera::validate (types.cpp:44-63) without a context or device (loaders,
 * load_camera_json): GVR_OK or GVR_ERR_VALIDATION with the message in msg. */
int gvr_camera_validate(const gvr_camera* camera, char* msg, int32_t msg_cap);
/* Profiling hook (no reference counterpart): while on, renders record the SM
 * cycles of each tile's selection CTA on the tape; read with gvr_tape_tile_cycles. */
int gvr_context_set_tile_profile(gvr_context* ctx, int on);
/* Per-tile selection cycles of a render made with the tile profile on
 * (n = tiles_x * tiles_y of the tape; 0 for tiles with nothing to select). */
int gvr_tape_tile_cycles(gvr_context* ctx, const gvr_tape* tape, int64_t* cycles, int64_t n);
/* Test hook: caps the tile-list pool and the backward's mask rectangles at `cap`
 * entries (8 B each; 0 = automatic sizing). Lists that do not fit stream every
 * kernel through the same exact tests (slower, same selection); kernels without a
 * mask rectangle take the backward's atomic fallback (same gradients within
 * rounding, not bit-deterministic). A small value exercises both paths in tests. */
int gvr_context_set_tile_capacity(gvr_context* ctx, int cap);
/* Test hook: tile lists longer than n entries (default and maximum 2048) are
 * sorted in global memory instead of shared memory. Results must not change. */
int gvr_context_set_list_smem(gvr_context* ctx, int n);

/* ---- CUDA graphs ----------------------------------------------------------
 * Capture a sequence of calls on the context stream (e.g. gvr_render +
 * gvr_scalar_loss + gvr_backward with DEVICE pointers, after one uncaptured
 * call has sized every buffer) and replay it with one launch. Calls that need
 * a host synchronisation (host outputs, scene upload) fail while capturing. */
int gvr_graph_begin(gvr_context* ctx);
int gvr_graph_end(gvr_context* ctx, gvr_graph** out);
int gvr_graph_launch(gvr_context* ctx, gvr_graph* graph);
void gvr_graph_destroy(gvr_graph* graph);

/* ---- scene: device-resident, validated once per upload ------------------ */
int gvr_scene_create(gvr_context* ctx, gvr_scene** out);
void gvr_scene_destroy(gvr_scene* scene);
/* Upload + validate (GaussianScene::validate, types.cpp:31-42). attr may be NULL when D == 0. */
int gvr_scene_set(gvr_context* ctx, gvr_scene* scene, int32_t K, int32_t D, double tau,
                  const double* centers, const double* inv_cov, const double* attr);
/* Same upload without the host synchronisation (fitting loops, graph capture):
 * the validation runs on the device and its result is read by gvr_scene_check
 * (the first error, with the gvr_scene_set message). Renders in between use the
 * uploaded values as they are. Capturable when the scene buffers already have
 * the size (one uncaptured call first) and the arrays are device pointers. */
int gvr_scene_set_deferred(gvr_context* ctx, gvr_scene* scene, int32_t K, int32_t D, double tau,
                           const double* centers, const double* inv_cov, const double* attr);
/* Result of the last gvr_scene_set_deferred (synchronises; re-read on every call,
 * so a captured upload is re-validated by every replay; GVR_OK after gvr_scene_set). */
int gvr_scene_check(gvr_context* ctx, gvr_scene* scene);
int32_t gvr_scene_size(const gvr_scene* scene);
int32_t gvr_scene_attr_dim(const gvr_scene* scene);

/* ---- forward ------------------------------------------------------------- */
int gvr_tape_create(gvr_context* ctx, gvr_tape** out);
void gvr_tape_destroy(gvr_tape* tape);

/* render_with_tape: view transform, projection + culling, 8x8 tile binning
 * (count pass, scan, emit), trace / top-K' selection, closed-form blend. The tape records the
 * per-pixel selection for gvr_backward and references `scene`, which must not be
 * re-set before the backward (checked). `out` may be NULL. */
int gvr_render(gvr_context* ctx, const gvr_scene* scene, const gvr_camera* camera,
               const gvr_selection* cfg, gvr_tape* tape, const gvr_render_outputs* out);

/* Tile-sharded render (C4: one large view split across GPUs): only tiles with
 * tile_index % nshards == shard are rendered; every other pixel gets the
 * empty-render outputs (0) and count 0, so the union over shards equals the
 * full render bit for bit, and gvr_backward on a shard tape yields that
 * shard's partial gradients (sum them across ranks). gvr_render = shard 0 of 1. */
int gvr_render_shard(gvr_context* ctx, const gvr_scene* scene, const gvr_camera* camera,
                     const gvr_selection* cfg, gvr_tape* tape, const gvr_render_outputs* out,
                     int32_t shard, int32_t nshards);

/* Copy out the taped selection (Tape::traced, grad.hpp:32): per pixel the selected
 * kernels ascending by (l, idx) with their FP64 (l, q, sigma); -1 / 0 padded.
 * Any pointer may be NULL. */
int gvr_tape_traced(gvr_context* ctx, const gvr_tape* tape, int32_t* idx, double* l, double* q,
                    double* sigma);
/* Tape::cam_scene (grad.hpp:29): the camera-space scene of the taped render
 * (view_transform, scene.cpp:5-17; centers K*3, inv_cov K*9; either nullable). */
int gvr_tape_cam_scene(gvr_context* ctx, const gvr_tape* tape, double* centers, double* inv_cov);
/* PixelKernelMap::dropped_behind_camera (tracer.hpp:39): kernels of the taped
 * render with camera-space z <= 1e-4. Synchronises. */
int gvr_tape_dropped_behind_camera(gvr_context* ctx, const gvr_tape* tape, int32_t* count);
/* validate_finite (blender.cpp:132-134) for a render whose outputs stayed on the
 * device: GVR_ERR_VALIDATION "image contains non-finite values" when any image,
 * alpha or depth value of the taped render is not finite. Synchronises. */
int gvr_tape_check_finite(gvr_context* ctx, gvr_tape* tape);
/* Tile-list layout of the taped render (no reference counterpart; synchronises):
 * stats[0] listed (tile, kernel) entries, [1] longest tile list, [2] tiles whose
 * list did not fit the pool (streamed: every kernel, no early exit), [3] lists
 * longer than the shared-memory stage (sorted in global memory), [4] pool capacity,
 * [5] backward mask-rectangle tiles requested, [6] mask capacity (kernels beyond it
 * take the non-deterministic atomic fallback). */
int gvr_tape_list_stats(gvr_context* ctx, const gvr_tape* tape, int64_t* stats);
/* Shape of the taped render. */
int gvr_tape_shape(const gvr_tape* tape, int32_t* height, int32_t* width, int32_t* k_prime,
                   int32_t* attr_dim);

/* ---- loss + backward ----------------------------------------------------- */
/* ScalarLoss::value on the taped render (grad.cpp:201-216). targets: H*W*max(D,1)
 * and H*W. loss_out (host or device, nullable). The upstream gradients are kept
 * in the tape for gvr_backward(d_image = NULL) and also written to
 * d_image_out / d_alpha_out when non-NULL. */
int gvr_scalar_loss(gvr_context* ctx, gvr_tape* tape, const double* target_image,
                    const double* target_alpha, double w_image, double w_alpha, double* loss_out,
                    double* d_image_out, double* d_alpha_out);

/* backward (grad.cpp:49-199). d_image: H*W*D, d_alpha: H*W; both NULL = use the
 * upstream stored by gvr_scalar_loss. flags NULL = both paths on. */
int gvr_backward(gvr_context* ctx, gvr_tape* tape, const double* d_image, const double* d_alpha,
                 const gvr_grad_flags* flags, const gvr_gradients* out);

/* As gvr_backward but ADDS the gradients into the (device) outputs: the
 * per-view accumulation of the fitting loop (fit.cpp:128-156). */
int gvr_backward_accumulate(gvr_context* ctx, gvr_tape* tape, const double* d_image, const double* d_alpha,
                            const gvr_grad_flags* flags, const gvr_gradients* out);

/* As gvr_backward, with the per-kernel gradients written as one DEVICE row per
 * kernel, packed[K*(9+D)] = [d_center(3) | d_inv_cov upper triangle (00 01 02 11
 * 12 22) | d_attr(D)], and d_rt[12] = [d_rotation(9) | d_translation(3)] (device):
 * the layout a multi-GPU reduction sums (tile-sharded C4: one reduce-scatter of
 * 9+D doubles per kernel instead of 15). */
int gvr_backward_packed(gvr_context* ctx, gvr_tape* tape, const double* d_image, const double* d_alpha,
                        const gvr_grad_flags* flags, double* packed, double* d_rt);

/* ---- fitting helpers ------------------------------------------------------ */
/* AdamState::update (fit.cpp:20-42) on arrays of n parameters (device, or host:
 * staged and copied back, synchronising); `step` is the 1-based step count used
 * for the bias corrections. */
int gvr_adam_step(gvr_context* ctx, double* params, const double* grads, double* m, double* v, int64_t n,
                  int64_t step, double lr, double beta1, double beta2, double eps);

/* As gvr_adam_step, with fit_shape's divergence rule (fit.cpp:246-250): when the
 * device scalar *loss is not finite, or *diverged is already set, nothing is
 * updated and *diverged (device int32) is set to 1. */
int gvr_adam_step_guarded(gvr_context* ctx, double* params, const double* grads, double* m, double* v, int64_t n,
                          int64_t step, double lr, double beta1, double beta2, double eps, const double* loss,
                          int32_t* diverged);

/* ---- sampler and render-path helpers -------------------------------------- */
/* gvr::sample_attributes (sampler.hpp:23-25, sampler.cpp:11-51): render (as
 * gvr_render), then per kernel alpha_k = sum_p W_pk obs_p / sum_p W_pk using the
 * rendering weights (normalized != 0: W / max(sum_p W, 1e-8) per pixel);
 * kernels with support < 1e-8 get zero attributes and masked = 1.
 * observed: obs_height*obs_width*channels; must match the camera size
 * (GVR_ERR_VALIDATION "observed image size does not match the camera").
 * Outputs attrs[K*channels], support[K], masked[K] (host or device, nullable). */
int gvr_sample_attributes(gvr_context* ctx, const gvr_scene* scene, const gvr_camera* camera,
                          const gvr_selection* cfg, const double* observed, int32_t obs_height, int32_t obs_width,
                          int32_t channels, int32_t normalized, double* attrs, double* support, uint8_t* masked);
/* The same on an existing taped render (the weights of gvr_render on that tape). */
int gvr_tape_sample_attributes(gvr_context* ctx, const gvr_tape* tape, const double* observed, int32_t channels,
                               int32_t normalized, double* attrs, double* support, uint8_t* masked);
/* gvr::resynthesize (sampler.cpp:53-66), scene part: dst = src with attributes
 * replaced by attrs[n_attrs*channels] (masked[k] != 0 -> zero; masked nullable),
 * validated like a render would. n_attrs != K -> GVR_ERR_VALIDATION
 * "sampled attribute count does not match the scene". Render dst to finish. */
int gvr_scene_resynthesize(gvr_context* ctx, gvr_scene* dst, const gvr_scene* src, int32_t n_attrs, int32_t channels,
                           const double* attrs, const uint8_t* masked);
/* gvr::transmittance_at (blender.hpp:29, blender.cpp:19-25) for every pixel of a
 * taped render: T(t[p]) over the pixel's selected kernels; t, out: H*W. */
int gvr_tape_transmittance(gvr_context* ctx, const gvr_tape* tape, const double* t, double* out);
/* gvr::normalized_weights (blender.hpp:36, blender.cpp:55-62) for every pixel:
 * out[H*W*k_prime] = W_k / max(sum W, eps), ascending (l, idx), 0 padded. */
int gvr_tape_normalized_weights(gvr_context* ctx, const gvr_tape* tape, double eps, double* out);
/* gvr::shade_lambert (blender.hpp:46-47, blender.cpp:146-172): normals H*W*3,
 * alpha/depth H*W (camera size), light_pos/light_color host double[3], out H*W*3. */
int gvr_shade_lambert(gvr_context* ctx, const gvr_camera* camera, const double* normals, const double* alpha,
                      const double* depth, const double* light_pos, const double* light_color, double* out);

/* ---- multi-view batches (C3 view-sharded renders, C5 fitting) ------------- */
/* n_views independent renders of one scene (SURVEY.md §8b "batched variants
 * over V cameras"): view v uses cameras[v], tapes[v] (distinct tapes) and
 * outs[v] (outs nullable). The views run concurrently on internal worker
 * streams forked from and joined into the context stream (graph-capturable). */
int gvr_render_views(gvr_context* ctx, const gvr_scene* scene, int32_t n_views, const gvr_camera* cameras,
                     const gvr_selection* cfg, gvr_tape* const* tapes, const gvr_render_outputs* outs);
/* ScalarLoss of every view against its own targets; losses[n_views] nullable. */
int gvr_scalar_loss_views(gvr_context* ctx, int32_t n_views, gvr_tape* const* tapes, const double* const* target_images,
                          const double* const* target_alphas, double w_image, double w_alpha, double* losses);
/* Backward of every view from the upstream stored by gvr_scalar_loss_views.
 * outs[n_views] (per-view bundles) and / or sum (+= the sum over views, views
 * added in ascending order) — DEVICE pointers, either nullable. */
int gvr_backward_views(gvr_context* ctx, int32_t n_views, gvr_tape* const* tapes, const gvr_grad_flags* flags,
                       const gvr_gradients* outs, const gvr_gradients* sum);

/* ---- fitting regularizers (fit.hpp:50-67, fit.cpp:44-115) ----------------- */
/* ShapeRegularizer::make: host edges[2*n_edges] (vertex pairs), rest_centers[3*n_vertices]
 * (host or device). No edges -> GVR_ERR_VALIDATION "regularizer needs a non-empty neighbor graph". */
int gvr_regularizer_create(gvr_context* ctx, int32_t n_vertices, int32_t n_edges, const int32_t* edges,
                           const double* rest_centers, gvr_regularizer** out);
void gvr_regularizer_destroy(gvr_regularizer* reg);
/* edge_reg / laplacian_reg at centers[3N]: *value = the (unweighted) term;
 * grad[3N] (nullable, host or device) receives weight * d(term)/d(centers),
 * added when accumulate != 0 (the fit loop's gradient), else overwritten. */
int gvr_edge_reg(gvr_context* ctx, const gvr_regularizer* reg, const double* centers, double weight, double* value,
                 double* grad, int32_t accumulate);
int gvr_laplacian_reg(gvr_context* ctx, const gvr_regularizer* reg, const double* centers, double weight,
                      double* value, double* grad, int32_t accumulate);

/* ---- building blocks of the reference API (C++ drop-in, include/gvr/) ------
 * One device launch per call; all pointers host or device; synchronising. */
/* trace_kernel (tracer.hpp:45, tracer.cpp:20-35) for n (ray, kernel) pairs:
 * dirs[n*3], centers[n*3], inv_cov[n*9] -> l, q, sigma [n] (nullable), bit-exact.
 * GVR_ERR_VALIDATION "trace_kernel: D^T inv_cov D <= 0 (inv_cov not positive-definite)". */
int gvr_trace_pairs(gvr_context* ctx, int64_t n, const double* dirs, const double* centers, const double* inv_cov,
                    double* l, double* q, double* sigma);
/* view_transform (scene.hpp:10, scene.cpp:5-17): camera validated first; bit-exact. */
int gvr_view_transform(gvr_context* ctx, int32_t K, const double* centers, const double* inv_cov,
                       const gvr_camera* camera, double* out_centers, double* out_inv_cov);
/* pixel_ray / generate_rays (scene.hpp:13-16, scene.cpp:19-33): dirs[n*3] of the
 * pixels (rows[i], cols[i]), or of every pixel row-major when rows == cols == NULL
 * (n = height * width). */
int gvr_pixel_rays(gvr_context* ctx, const gvr_camera* camera, int64_t n, const int32_t* rows, const int32_t* cols,
                   double* dirs);
/* coarse_select (tracer.hpp:49, tracer.cpp:37-113) on a camera-space scene: per
 * kernel the pixel box it is pushed into, boxes[K*4] = {row_lo, row_hi, col_lo,
 * col_hi} ({1, 0, 1, 0} = not pushed), and PixelKernelMap::dropped_behind_camera;
 * the cells (ds x ds) of the box are the kernel's cells. Config validated first. */
int gvr_coarse_select_boxes(gvr_context* ctx, int32_t K, const double* cam_centers, const double* cam_inv_cov,
                            const gvr_camera* camera, const gvr_selection* cfg, int32_t* boxes, int32_t* dropped);
/* fine_select / blend order (tracer.cpp:115-127): the entries with q > ln(eta)
 * (all when eta is outside (0, 1)) sorted by (l, idx); order[m] = input positions.
 * n <= 2048 per call. */
int gvr_ray_sort(gvr_context* ctx, int32_t n, const int32_t* idx, const double* l, const double* q, double eta,
                 int32_t* order, int32_t* m_out);
/* blend (blender.hpp:33, blender.cpp:27-53) of one ray (n <= 2048): weights in
 * ascending (l, idx) order (out_idx, out_w [n]) and alpha (FP64 erfc / exp). */
int gvr_blend_ray(gvr_context* ctx, int32_t n, const int32_t* idx, const double* l, const double* q,
                  const double* sigma, double tau, int32_t* out_idx, double* out_w, double* alpha);
/* transmittance_at (blender.hpp:29, blender.cpp:19-25) of one ray's entries at nt depths. */
int gvr_transmittance_ray(gvr_context* ctx, int32_t n, const double* l, const double* q, const double* sigma,
                          double tau, int32_t nt, const double* t, double* out);
/* normalized_weights (blender.hpp:36, blender.cpp:55-62): w / max(sum w, eps). */
int gvr_normalized_weights_ray(gvr_context* ctx, int32_t n, const double* w, double eps, double* out);
/* ScalarLoss::value (grad.hpp:68, grad.cpp:201-216) on caller buffers:
 * loss = sum w_i (x - t)^2 / 2 over image then alpha; d_image / d_alpha nullable. */
int gvr_scalar_loss_buffers(gvr_context* ctx, int64_t n_img, const double* image, const double* target_image,
                            int64_t n_alpha, const double* alpha, const double* target_alpha, double w_image,
                            double w_alpha, double* loss, double* d_image, double* d_alpha);

#ifdef __cplusplus
}
#endif
#endif /* GVR_CUDA_H */
