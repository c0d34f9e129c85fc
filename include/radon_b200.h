/*
 * radon_b200.h — C ABI of the B200-native (sm_100a) Radon projector.
 *
 * Drop-in replacement for the hot path of the reference ("radonkit", the CPU
 * restatement of TorchRadon, /root/reference/proj/core):
 *
 *   reference entry point                                   replaced by
 *   -----------------------------------------------------   ---------------------------
 *   make_parallel / make_fanbeam   geometry.hpp:38-48        rk_geometry_resolve
 *   angles_linspace                geometry.hpp:54           rk_angles_linspace
 *   forward(geom, image, opts)     projector.hpp:19-21       rk_forward / rk_forward_host
 *   backprojection(geom, sino, ..) projector.hpp:27-29       rk_backproject / rk_backproject_host
 *   make_filter(kind, det_count)   sino_filter.hpp:30-31     rk_filter_create / rk_filter_response
 *   filter_kind_from_name          sino_filter.hpp:14        rk_filter_kind_from_name
 *   filter_sinogram(sino, filter)  sino_filter.hpp:36        rk_filter_sinogram / _host
 *   fbp(geom, sino, kind)          sino_filter.hpp:39-41     rk_fbp / rk_fbp_host
 *   projector_operator(geom).apply/.adjoint  linop.cpp:33-41 rk_forward / rk_backproject
 *   landweber / estimate_alpha / cgne  solvers.hpp:14-31     rk_landweber / rk_estimate_alpha / rk_cgne
 *
 * Conventions are the reference's (geometry.hpp:10-16): image B x s x s
 * row-major (row 0 at the top), sinogram B x n_angles x det_count, angles in
 * radians, detector cell k at u_k = (k - det_count/2 + 0.5) * det_spacing.
 *
 * Storage dtypes RK_F16 / RK_F32 / RK_F64; arithmetic is fp32 throughout
 * (north star); the output keeps the input's storage dtype, like the
 * reference (projector.cpp:207-224).  fp16 narrowing is round-to-nearest-even
 * and unchecked (overflow -> inf), as Tensor::from_double_as (tensor.cpp:121).
 *
 * Every function returns an rk_status; on failure rk_last_error() (thread
 * local) holds the message.  Status codes mirror the reference's exception
 * taxonomy (errors.hpp:9-40, CLI exit codes cli.cpp:718-730).
 *
 * Device entry points take device pointers and a cudaStream_t (as void*,
 * NULL = legacy default stream) and are asynchronous.  *_host entry points
 * take host buffers (pinned for full speed), are synchronous and return
 * results in host memory — the exact semantics of the reference's
 * Tensor-in / Tensor-out functions.
 *
 * Results are deterministic: every output element is a fixed-order
 * reduction independent of batch size, grid shape and GPU count (the
 * reference's batch- and thread-invariance contract, threading.hpp:12-15,
 * acceptance.cpp:340-389).
 */
#ifndef RADON_B200_H_
#define RADON_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RK_VERSION_MAJOR 0
#define RK_VERSION_MINOR 1

typedef enum {
  RK_OK = 0,
  RK_ERR_VALIDATION = 1, /* ValidationError (errors.hpp:9-13)              */
  RK_ERR_NUMERICAL = 2,  /* NumericalError family (errors.hpp:16-40)       */
  RK_ERR_CUDA = 3        /* CUDA runtime failure (no reference equivalent) */
} rk_status;

typedef enum { RK_F16 = 0, RK_F32 = 1, RK_F64 = 2 } rk_dtype; /* Precision::{Half,Single,Double} */

typedef enum { RK_PARALLEL = 0, RK_FANBEAM = 1 } rk_geometry_kind;

typedef enum { /* FilterKind, sino_filter.hpp:12 */
               RK_RAM_LAK = 0,
               RK_SHEPP_LOGAN = 1,
               RK_COSINE = 2,
               RK_HAMMING = 3,
               RK_HANN = 4
} rk_filter_kind;

/* Optional-field flags: an unset flag means "use the reference default"
 * (the std::optional arguments of make_parallel / make_fanbeam). */
#define RK_HAS_DET_COUNT 0x1u
#define RK_HAS_DET_SPACING 0x2u
#define RK_HAS_DET_DISTANCE 0x4u

typedef struct rk_geometry {
  int32_t kind;           /* rk_geometry_kind                                   */
  uint32_t has;           /* RK_HAS_* flags                                     */
  int64_t image_size;     /* s: image is s x s                                  */
  int64_t n_angles;       /* number of projection angles                        */
  const double* angles;   /* n_angles radians (copied by rk_plan_create)        */
  int64_t det_count;      /* default: image_size                                */
  double det_spacing;     /* default: 1 (parallel), magnification*s/nd (fan)    */
  double source_distance; /* fan-beam only                                      */
  double det_distance;    /* fan-beam only, default: source_distance            */
  double step;            /* ProjectorOptions::step (projector.hpp:8-11), > 0   */
} rk_geometry;

typedef struct rk_plan rk_plan;
typedef struct rk_filter rk_filter;

typedef struct rk_plan_info {
  rk_geometry geometry;         /* resolved (defaults applied, has = all flags)        */
  int64_t forward_samples;      /* exact sum over rays of max(1, ceil(len/step))       */
  int64_t backproject_samples;  /* s * s * n_angles                                    */
  int32_t device;               /* CUDA device the plan lives on                       */
  int32_t flags;                /* RK_PLAN_* bits below                                */
} rk_plan_info;

/* rk_plan_info.flags */
#define RK_PLAN_SCHEDULED 1       /* the forward schedule exists (first forward / rk_plan_prepare done) */
#define RK_PLAN_SCHEDULE_CACHED 2 /* ... and came from the on-disk plan cache ($RK_PLAN_CACHE)          */

/* ------------------------------------------------------------- misc */
const char* rk_last_error(void);
const char* rk_version(void);

/* ------------------------------------------------------------- geometry */
/* Applies the make_parallel / make_fanbeam defaults and validation
 * (geometry.cpp:22-55); `out->angles` aliases `in->angles`. */
int rk_geometry_resolve(const rk_geometry* in, rk_geometry* out);
/* n evenly spaced angles on [start, stop) (geometry.cpp:67-73). */
int rk_angles_linspace(double start, double stop, int64_t n, double* out);

/* ------------------------------------------------------------- plans */
/* Validates + resolves the geometry, builds the per-angle and per-ray
 * tables on `device` (fp64 ray setup, projector.cpp:37-139).  device -1
 * builds a host-only plan (tables and work counts, no kernels). */
int rk_plan_create(const rk_geometry* geometry, int device, rk_plan** plan);
int rk_plan_destroy(rk_plan* plan);
int rk_plan_info_get(const rk_plan* plan, rk_plan_info* info);
/* Builds (or loads from the plan cache) the forward schedule now instead of on
 * the first rk_forward — the planning the reference's stateless forward
 * (projector.cpp:228-236) never pays; `hash` (optional) receives a 64-bit
 * FNV-1a digest of the schedule tables (equal digests = identical launches). */
int rk_plan_prepare(rk_plan* plan, uint64_t* hash);

/* ------------------------------------------------------------- projector */
/* Any batch >= 1: beyond 262,140 images (65,535 packed groups, one launch's
 * grid limit) the device calls run consecutive sub-batches, bit-identical per
 * image (rk_forward, rk_backproject, rk_filter_sinogram, rk_fbp and the *_host
 * calls); the solvers and ADMM keep whole-batch state and return
 * RK_ERR_VALIDATION above that batch. */
/* image: batch x s x s (dtype) -> sino: batch x n_angles x det_count (dtype). */
int rk_forward(rk_plan* plan, int dtype, const void* d_image, int64_t batch, void* d_sino, void* stream);
/* sino: batch x n_angles x det_count -> image: batch x s x s. */
int rk_backproject(rk_plan* plan, int dtype, const void* d_sino, int64_t batch, void* d_image, void* stream);

/* ------------------------------------------------------------- filter */
int rk_filter_kind_from_name(const char* name, int* kind);
const char* rk_filter_kind_name(int kind);
/* Ramp response of make_filter (sino_filter.cpp:64-92), uploaded to `device`
 * (device -1: host-only, for inspecting the response without a GPU).
 * det_count 2 .. 16384 (padded transforms up to 2^15 points; above 2^13 the
 * filter runs on two-CTA clusters). */
int rk_filter_create(int kind, int64_t det_count, int device, rk_filter** filter);
int rk_filter_destroy(rk_filter* filter);
/* Host copy of the response: padded size, padded/2+1 double and float bins
 * (either pointer may be NULL). */
int rk_filter_response(const rk_filter* filter, int64_t* padded_size, double* response, float* response_f);
/* sino: batch x n_angles x det_count -> same shape (sino_filter.cpp:98-124). */
int rk_filter_sinogram(rk_filter* filter, int dtype, const void* d_in, int64_t batch, int64_t n_angles,
                       void* d_out, void* stream);
/* backprojection(filter_sinogram(sino)) (sino_filter.cpp:126-136); the
 * filtered sinogram lives in plan scratch. */
int rk_fbp(rk_plan* plan, rk_filter* filter, int dtype, const void* d_sino, int64_t batch, void* d_image,
           void* stream);

/* ------------------------------------------------------------- host-buffer (reference-shaped) calls */
/* Synchronous; copies are pipelined against the kernels in batch chunks. */
int rk_forward_host(rk_plan* plan, int dtype, const void* h_image, int64_t batch, void* h_sino);
int rk_backproject_host(rk_plan* plan, int dtype, const void* h_sino, int64_t batch, void* h_image);
int rk_filter_sinogram_host(rk_filter* filter, int dtype, const void* h_in, int64_t batch, int64_t n_angles,
                            void* h_out);
int rk_fbp_host(rk_plan* plan, rk_filter* filter, int dtype, const void* h_sino, int64_t batch, void* h_image);

/* ------------------------------------------------------------- solvers (config 5) */
/* alpha = 2 / sigma_max^2 of A'A by `iterations` power iterations from the
 * reference's seeded uniform start vector (solvers.cpp:111-128). */
int rk_estimate_alpha(rk_plan* plan, int iterations, uint64_t seed, double* alpha);
/* x <- x - alpha * A'(Ax - y), `iterations` times, fp32 state
 * (solvers.cpp:130-145).  Returns RK_ERR_NUMERICAL (DivergenceError) when an
 * iterate becomes non-finite; *failed_iteration receives the iteration. */
int rk_landweber(rk_plan* plan, int dtype, const void* d_y, const void* d_guess, int64_t batch, double alpha,
                 int iterations, void* d_x, int* failed_iteration, void* stream);
/* CG on A'A x = A'y with per-element fp64 scalars and freeze-on-tolerance
 * (solvers.cpp:47-107,162-166).  RK_ERR_NUMERICAL on non-positive curvature
 * (NotPositiveDefiniteError). */
int rk_cgne(rk_plan* plan, int dtype, const void* d_y, const void* d_guess, int64_t batch, int max_iter,
            double tolerance, void* d_x, int* failed_iteration, void* stream);

/* ------------------------------------------------------------- shearlets + ADMM */
typedef struct rk_shearlet rk_shearlet;
/* make_plan (shearlet.hpp:37): cone-adapted alpha-shearlet Fourier multipliers,
 * Parseval-normalised; any square grid >= 2 (<= 8192) on the device: radix-2
 * shared-memory FFTs for powers of two, DFT-matrix transforms otherwise.
 * device -1: host-only (multipliers for inspection). */
int rk_shearlet_create(int64_t height, int64_t width, const double* alphas, int n_scales, int device,
                       rk_shearlet** plan);
/* make_plan_cached (shearlet.hpp:43, shearlet.cpp:201-249): a plan over stored
 * n_coeff x h x w fp64 multipliers (the cache file's payload), used verbatim. */
int rk_shearlet_create_stored(int64_t height, int64_t width, const double* alphas, int n_scales,
                              const double* multipliers, int device, rk_shearlet** plan);
int rk_shearlet_destroy(rk_shearlet* plan);
/* n_coeff; scales (n_coeff labels, may be NULL); multipliers (n_coeff x h x w fp64, may be NULL). */
int rk_shearlet_info(const rk_shearlet* plan, int64_t* n_coeff, double* scales, double* multipliers);
/* forward(plan, image): batch x h x w -> batch x n_coeff x h x w (shearlet.hpp:49). */
int rk_shearlet_forward(rk_shearlet* plan, int dtype, const void* d_image, int64_t batch, void* d_coeff,
                        void* stream);
/* backward(plan, coeff): batch x n_coeff x h x w -> batch x h x w, exact adjoint (shearlet.hpp:51). */
int rk_shearlet_backward(rk_shearlet* plan, int dtype, const void* d_coeff, int64_t batch, void* d_image,
                         void* stream);

/* admm_reconstruct (admm.hpp:49-50, admm.cpp:111-163): l1-shearlet ADMM with a
 * positivity split; CG on (p0 A'A + (1 + p1) I) warm-started from the previous
 * f, `inner_cg_iterations` steps per outer iteration.  weights: n_coeff values,
 * NULL = 3^scale / 400 (admm.cpp:11-15).  fp32 state for every storage dtype.
 * The shearlet grid must equal the projector's image grid.  A non-finite state
 * returns RK_ERR_NUMERICAL (DivergenceError) with *failed_iteration set. */
int rk_admm(rk_plan* plan, rk_shearlet* shearlet, int dtype, const void* d_sino, int64_t batch, double p0, double p1,
            const double* weights, int64_t outer_iterations, int inner_cg_iterations, void* d_image,
            int64_t* failed_iteration, void* stream);
/* Stepwise form (the reference's AdmmObserver, admm.hpp:33-34): create computes
 * bp = A'y and the zero state; iterate runs n outer iterations; read copies one
 * state variable (0 f, 1 z1, 2 u1, 3 z2, 4 u2; f/z2/u2 batch x h x w, z1/u1
 * batch x n_coeff x h x w) into device memory in `dtype`. */
typedef struct rk_admm_state rk_admm_state;
int rk_admm_create(rk_plan* plan, rk_shearlet* shearlet, int dtype, const void* d_sino, int64_t batch, double p0,
                   double p1, const double* weights, int inner_cg_iterations, void* stream, rk_admm_state** admm);
int rk_admm_iterate(rk_admm_state* admm, int64_t n, int64_t* failed_iteration, void* stream);
int rk_admm_read(rk_admm_state* admm, int which, int dtype, void* d_dst, void* stream);
int rk_admm_destroy(rk_admm_state* admm);

/* ------------------------------------------------------------- instrumentation (no reference equivalent) */
typedef enum {
  RK_KERNEL_PACK = 0,        /* layout packing (image / sinogram -> 4-image interleave) */
  RK_KERNEL_FORWARD = 1,     /* ray-driven forward projector                             */
  RK_KERNEL_BACKPROJECT = 2, /* pixel-driven backprojector                               */
  RK_KERNEL_FILTER = 3,      /* ramp filter                                              */
  RK_KERNEL_SOLVER = 4,      /* fused solver vector kernels / reductions                 */
  RK_KERNEL_SHEARLET = 5,    /* shearlet 2-D FFT passes / ADMM updates                    */
  RK_KERNEL_KINDS = 6
} rk_kernel_kind;

typedef struct rk_kernel_stats {
  int64_t launches[RK_KERNEL_KINDS]; /* kernels launched since the last reset           */
  int64_t timed[RK_KERNEL_KINDS];    /* of which bracketed by events (profiling enabled) */
  double ms[RK_KERNEL_KINDS];        /* summed device time of the timed launches         */
} rk_kernel_stats;

/* Bracket every subsequent kernel launch with CUDA events on its stream. */
int rk_profiling_enable(int enable);
/* Synchronises on the recorded events and returns the totals; reset != 0
 * clears counters and records. */
int rk_profiling_read(rk_kernel_stats* stats, int reset);
/* Measured shared-memory (LDS.128) bandwidth of `device` in GB/s: the
 * L1TEX/SMEM roofline peak of the projector kernels. */
int rk_probe_smem_bandwidth(int device, double* gbs);

#ifdef __cplusplus
}
#endif

#endif /* RADON_B200_H_ */
