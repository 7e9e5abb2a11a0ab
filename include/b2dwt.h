/*
 * b2dwt.h -- C ABI of the B200-native 2-D DWT hot path (libb2dwt.so).
 *
 * Drop-in boundary for the reference's pixel executor (liftfuse, Python):
 *
 *   b2dwt_plan_create     <- liftfuse.engine.compile_scheme() output consumed by
 *                            run_tiled(program, comps, cfg)     engine.py:404-439
 *                            (a b2dwt_program is a StencilProgram flattened,
 *                             engine.py:227-256, terms in compiled order :267)
 *   b2dwt_run_components  <- run_tiled / run_reference on 4 component planes
 *                            engine.py:404-439, :442-451
 *   b2dwt_forward         <- forward(image, scheme, cfg): deinterleave + run_tiled
 *                            engine.py:481-487, deinterleave :200-211 (fused)
 *   b2dwt_inverse         <- inverse(quad, scheme, cfg): run_tiled + interleave_quad
 *                            engine.py:490-495, interleave_quad :214-221 (fused)
 *   b2dwt_forward_rows    <- forward() restricted to a band of output rows of a
 *                            larger image (multi-GPU row strips; new, no reference
 *                            counterpart; reflection stays in global coordinates)
 *   b2dwt_inverse_rows    <- inverse() restricted to a band of output rows (new)
 *   b2dwt_dwt / b2dwt_idwt<- multi-level pyramid (new; oracle = forward iterated
 *                            on ll)
 *   b2dwt_forward2        <- two levels of that pyramid in one kernel (new)
 *   b2dwt_dwt_host /      <- the same pyramids from / to HOST arrays, as the
 *   b2dwt_idwt_host          reference's callers hold them (engine.py:481-495);
 *                            PCIe copies pipelined in row bands
 *   b2dwt_lift1d /        <- apply_plan_1d / invert_plan_1d, schemes.py:806-856
 *   b2dwt_unlift1d           (batched 1-D lifting)
 *
 * Conventions
 *   - All pixel pointers are DEVICE pointers owned by the caller (except the
 *     image / subband pointers of b2dwt_dwt_host and b2dwt_idwt_host, which
 *     are host pointers); element type is float (B2DWT_F32) or double
 *     (B2DWT_F64) as given at plan creation.
 *   - Leading dimensions (ld) and batch strides are in ELEMENTS.
 *   - Quad grid: an H x W image has rows = H/2, cols = W/2 quads; component 0..3
 *     = (even row, even col)=LL, (even, odd)=HL, (odd, even)=LH, (odd, odd)=HH
 *     (engine.py:52, schemes.py:3-14).
 *   - Boundary handling is the reference's whole-sample symmetric extension
 *     applied to the state entering every sub-step (engine.py:55-92, 312-347).
 *   - Calls are asynchronous on `stream` (a cudaStream_t, NULL = legacy default
 *     stream).  Plans are immutable and may be shared across threads.  The
 *     library's only process-wide state is internal and lock-protected: per-
 *     device caches (function attributes, SM counts) and zero-initialised
 *     work-split counters (a pool per stream -- launches ordered on a stream
 *     reuse them -- and a never-reused arena for launches captured into CUDA
 *     graphs, which may replay concurrently with anything).
 *   - Return 0 on success or a negative B2DWT_E* code; b2dwt_last_error()
 *     returns a thread-local message.  There is no CPU fallback: without a
 *     CUDA device every compute entry point fails with B2DWT_ECUDA.
 */
#ifndef B2DWT_H
#define B2DWT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B2DWT_ABI_VERSION 1

enum {
    B2DWT_OK = 0,
    B2DWT_EINVAL = -22,       /* bad argument (shape, pointer, layout)      */
    B2DWT_EUNSUPPORTED = -95, /* valid request this build cannot execute    */
    B2DWT_ECUDA = -5,         /* CUDA runtime error (message has details)   */
    B2DWT_ENOMEM = -12
};

enum { B2DWT_F32 = 0, B2DWT_F64 = 1 };

/* Plan flags */
enum {
    B2DWT_STRICT = 1,        /* bit-exact with the reference: every product and sum
                                rounded separately, in compiled term order (default) */
    B2DWT_FAST = 2,          /* fused multiply-add; within 1e-4 x input range (f32)  */
    B2DWT_FORCE_GENERIC = 4, /* use the per-sub-step interpreter kernel (debug)      */
    B2DWT_NO_TMA = 8,        /* fused kernel loads with cp.async instead of TMA      */
    B2DWT_NO_TILE = 16,      /* never use the 2-D tile kernel (small levels stream)  */
    B2DWT_FORCE_TILE = 32,   /* tile kernel for every whole-image level it supports  */
    B2DWT_NO_FUSE = 64       /* b2dwt_dwt: one launch per level (no two-level fused
                                kernel; results are identical either way)           */
};

/* One multiply-accumulate term: out[target][n,m] += coeff * in[src][n+dn, m+dm] */
typedef struct {
    int32_t src; /* 0..3 */
    int32_t dm;  /* column offset, quads */
    int32_t dn;  /* row offset, quads    */
    int32_t reserved;
    double coeff;
} b2dwt_term;

/* A StencilProgram (engine.py:247-256) with pass boundaries dropped: the
 * transform is the composition of its sub-steps, each a gather over the
 * previous sub-step's full output. */
typedef struct {
    int32_t abi_version;       /* B2DWT_ABI_VERSION */
    int32_t n_substeps;
    const int32_t* term_counts; /* [n_substeps * 4]: terms of (substep, target) */
    const b2dwt_term* terms;    /* flattened in (substep, target, term) order   */
} b2dwt_program;

typedef struct b2dwt_plan_s* b2dwt_plan;

typedef struct {
    int32_t kernel;        /* 0 = generic per-sub-step interpreter, 1 = fused streaming */
    int32_t program_id;    /* built-in structure index, -1 for generic                  */
    int32_t halo_left, halo_right, halo_up, halo_down; /* fused cone, quads            */
    int32_t dtype, flags;
    char key[64];          /* e.g. "cdf97/non-separable-split/fwd" or "generic"         */
} b2dwt_plan_info;

/* Four component planes in quad coordinates. */
typedef struct {
    void* ptr[4];
    int64_t ld[4];    /* elements between rows, per plane   */
    int64_t bstride;  /* elements between batch items (all planes) */
} b2dwt_planes;

int32_t b2dwt_abi_version(void);
const char* b2dwt_last_error(void);
/* Number of CUDA devices visible (0 on a CPU-only host); never fails. */
int32_t b2dwt_device_count(void);

int b2dwt_plan_create(const b2dwt_program* program, int32_t dtype, int32_t flags, b2dwt_plan* out);
int b2dwt_plan_destroy(b2dwt_plan plan);
int b2dwt_plan_get_info(b2dwt_plan plan, b2dwt_plan_info* info);

/* Components -> components (run_tiled). rows x cols quads, `batch` items. */
int b2dwt_run_components(b2dwt_plan plan, const b2dwt_planes* in, const b2dwt_planes* out,
                         int64_t rows, int64_t cols, int32_t batch, void* stream);

/* Interleaved image (height x width, even) -> 4 subband planes. */
int b2dwt_forward(b2dwt_plan plan, const void* image, int64_t image_ld, int64_t image_bstride,
                  int64_t height, int64_t width, const b2dwt_planes* out, int32_t batch, void* stream);

/* 4 subband planes -> interleaved image (height x width). `plan` holds the
 * INVERSE program (compile_scheme(invert_scheme(scheme))). */
int b2dwt_inverse(b2dwt_plan plan, const b2dwt_planes* in, void* image, int64_t image_ld,
                  int64_t image_bstride, int64_t height, int64_t width, int32_t batch, void* stream);

/* Row-band forward for row-strip decomposition.  The image is global_height x
 * width; `image` points at global pixel row `image_row0` (even) and holds
 * `image_rows` rows (even).  Computes quad rows [out_row_begin, out_row_end)
 * into `out` whose row 0 is quad row out_row_begin.  The buffer must hold the
 * fused cone: quad rows [out_row_begin - halo_up, out_row_end + halo_down)
 * clipped to the image (see b2dwt_plan_info).  Bit-identical to the same rows
 * of b2dwt_forward on the whole image. */
int b2dwt_forward_rows(b2dwt_plan plan, const void* image, int64_t image_ld, int64_t image_row0,
                       int64_t image_rows, int64_t global_height, int64_t width, int64_t out_row_begin,
                       int64_t out_row_end, const b2dwt_planes* out, void* stream);

/* Row-band inverse (the mirror of b2dwt_forward_rows; `plan` holds the inverse
 * program).  The four subband planes `in` hold quad rows [in_row0, in_row0 +
 * in_rows) of a global_height x width image's subbands (row 0 of each plane is
 * quad row in_row0); they must cover [out_row_begin - halo_up, out_row_end +
 * halo_down) clipped to the image.  Writes pixel rows [2*out_row_begin,
 * 2*out_row_end) to `image`, which points at pixel row 2*out_row_begin.
 * Bit-identical to the same rows of b2dwt_inverse on the whole image. */
int b2dwt_inverse_rows(b2dwt_plan plan, const b2dwt_planes* in, int64_t in_row0, int64_t in_rows, void* image,
                       int64_t image_ld, int64_t global_height, int64_t width, int64_t out_row_begin,
                       int64_t out_row_end, void* stream);

/* Multi-level forward pyramid.  Level l (0-based) transforms the (H>>l) x (W>>l)
 * LL of level l-1 (level 0: `image`).  details[l] receives HL/LH/HH of level l
 * (ptr[0] ignored); `ll_out` (pitch ll_ld) receives the final LL, an
 * (H >> levels) x (W >> levels) plane.  `scratch` must hold
 * (H/2)*(W/2) + (H/4)*(W/4) elements (LL ping-pong between levels, so no level
 * reads and writes the same buffer); it may be NULL when levels == 1.  H and W
 * must be divisible by 2^levels.  Batch = 1. */
int b2dwt_dwt(b2dwt_plan plan, const void* image, int64_t image_ld, int64_t height, int64_t width,
              int32_t levels, const b2dwt_planes* details, void* ll_out, int64_t ll_ld, void* scratch,
              void* stream);

/* Two pyramid levels in ONE kernel (new): level 0 of the height x width
 * `image` and level 1 of its LL, which never leaves the SM (the LL band of
 * level 0 is not written anywhere).  det0.ptr[1..3] receive level 0's HL/LH/HH
 * ((H/2) x (W/2)), out1.ptr[0..3] level 1's LL/HL/LH/HH ((H/4) x (W/4)).
 * Bit-identical to two b2dwt_forward calls.  Returns B2DWT_EUNSUPPORTED when
 * the plan or geometry does not fit the fused kernel (built-in forward lifting
 * program, f32, 16-B aligned image pitch, W >= 256, H and W divisible by 4, no
 * B2DWT_NO_FUSE / NO_TMA / FORCE_GENERIC flag); the caller then runs two
 * levels.  b2dwt_dwt pairs its levels this way automatically. */
int b2dwt_forward2(b2dwt_plan plan, const void* image, int64_t image_ld, int64_t height, int64_t width,
                   const b2dwt_planes* det0, const b2dwt_planes* out1, void* stream);

/* Multi-level inverse: `plan` holds the inverse program.  Reconstructs the
 * height x width image from ll (of the coarsest level) and details[l].
 * `scratch` as for b2dwt_dwt. */
int b2dwt_idwt(b2dwt_plan plan, const void* ll, int64_t ll_ld, const b2dwt_planes* details, int32_t levels,
               void* image, int64_t image_ld, int64_t height, int64_t width, void* scratch, void* stream);

/* Multi-level forward pyramid of a HOST image into HOST subbands (the
 * reference's host-array call, engine.py:481-487, iterated on LL), with the
 * PCIe traffic pipelined: the image is uploaded in `bands` row chunks on one
 * internal stream, every level is computed band by band (b2dwt_forward_rows)
 * on `stream` as soon as its input rows plus the cone exist, and each finished
 * band's HL/LH/HH rows (and the final LL) are downloaded on a second internal
 * stream while later bands are still uploading.  `details[l].ptr[1..3]` and
 * `ll_out` are host pointers (pinned memory gives the overlap; pageable memory
 * is correct but serialises the copies).  `workspace` is device memory of at
 * least b2dwt_dwt_host_workspace() bytes, 256-B aligned.  Asynchronous: the
 * outputs are complete once `stream` reaches the point of the call.  Needs a
 * fused built-in forward plan; bit-identical to b2dwt_dwt.  bands <= 0: 16. */
int64_t b2dwt_dwt_host_workspace(b2dwt_plan plan, int64_t height, int64_t width, int32_t levels);
int b2dwt_dwt_host(b2dwt_plan plan, const void* image, int64_t image_ld, int64_t height, int64_t width,
                   int32_t levels, const b2dwt_planes* details, void* ll_out, int64_t ll_ld, void* workspace,
                   int64_t workspace_bytes, int32_t bands, void* stream);

/* Multi-level inverse from HOST subbands into a HOST image (`plan` holds the
 * inverse program): the coarse levels are uploaded and inverted whole, level 0
 * runs in `bands` row bands with its upload, kernels and image download
 * overlapped.  Host pointers as for b2dwt_dwt_host; `workspace` holds
 * b2dwt_idwt_host_workspace() bytes.  Bit-identical to b2dwt_idwt. */
int64_t b2dwt_idwt_host_workspace(b2dwt_plan plan, int64_t height, int64_t width, int32_t levels);
int b2dwt_idwt_host(b2dwt_plan plan, const void* ll, int64_t ll_ld, const b2dwt_planes* details, int32_t levels,
                    void* image, int64_t image_ld, int64_t height, int64_t width, void* workspace,
                    int64_t workspace_bytes, int32_t bands, void* stream);

/* Batched 1-D lifting (schemes.py:806-856 apply_plan_1d / invert_plan_1d) on
 * `batch` signals of `length` (even) samples, row pitch *_ld in elements.
 * Steps are applied in order; step s updates the odd/high plane (target 1,
 * reading the even samples) or the even/low plane (target 0, reading the odd
 * samples) with step_count[s] terms (shift k, coefficient c) in ascending k:
 * x[i] += c * other[ext(i - k)], whole-sample symmetric extension.  Forward:
 * split, steps, then multiply by scale = {lo, hi} (NULL: none).  Inverse
 * (b2dwt_unlift1d, in place in low/high): divide by scale, the steps as given
 * (the caller passes them reversed and negated), then merge.  f64 is
 * bit-identical to the reference's Python floats. */
int b2dwt_lift1d(int32_t dtype, int32_t n_steps, const int32_t* step_target, const int32_t* step_count,
                 const int32_t* shifts, const double* coefs, const double* scale, const void* signal,
                 int64_t signal_ld, void* low, void* high, int64_t out_ld, int64_t length, int32_t batch,
                 void* stream);
int b2dwt_unlift1d(int32_t dtype, int32_t n_steps, const int32_t* step_target, const int32_t* step_count,
                   const int32_t* shifts, const double* coefs, const double* scale, void* low, void* high,
                   int64_t band_ld, void* signal, int64_t signal_ld, int64_t length, int32_t batch, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* B2DWT_H */
