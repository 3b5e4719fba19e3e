/*
 * ddm-b200 C-ABI: the drop-in boundary of the B200 WITH_FT (FFT-in-time) structure-function
 * path.  Plain pointers and sizes only; no exception or C++ type crosses it.  Every entry
 * point returns a status:
 *   0 ok, 1 input (ddm::InputError), 2 plan (ddm::PlanError, device memory), 3 io
 *   (ddm::IoError), 4 cuda (device failure), 5 internal;
 * and on failure ddm_b200_last_error() returns a thread-local message.
 *
 * The reference (`/root/reference/proj`) is a C++ library with no FFI of its own; each
 * entry point below names the reference interface it replaces (INTEGRATION.md shows the
 * ctypes / C++ bindings a maintainer would add).
 */
#ifndef DDM_B200_H
#define DDM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DDM_B200_OK 0
#define DDM_B200_E_INPUT 1
#define DDM_B200_E_PLAN 2
#define DDM_B200_E_IO 3
#define DDM_B200_E_CUDA 4
#define DDM_B200_E_INTERNAL 5

/* ddm::RunCounters (proj/core/include/ddm/timing.hpp:38-50) */
typedef struct ddm_b200_counters {
    uint64_t spatial_ffts;
    uint64_t temporal_ffts;
    uint64_t pairs;
} ddm_b200_counters;

/* ddm::TimingBreakdown (proj/core/include/ddm/timing.hpp:12-29), seconds */
typedef struct ddm_b200_timing {
    double disk, step1, step2, merge, other, total;
} ddm_b200_timing;

/* Called with the workspace path after partials are written, before the merge
   (ddm::RunConfig::before_merge, proj/core/include/ddm/scheduler.hpp:90-92). */
typedef void (*ddm_b200_before_merge_fn)(const char* workspace, void* user);

/* ddm::RunConfig (proj/core/include/ddm/scheduler.hpp:78-93) */
typedef struct ddm_b200_run_config {
    int algorithm;          /* 0 = with_ft (the only accelerated algorithm) */
    int precision;          /* 0 = f32, 1 = f64 */
    const int64_t* lags;    /* n_lags values, NULL/0 = every lag 0..N-1 */
    int64_t n_lags;
    int has_q_max;          /* optional<double> q_max */
    double q_max;
    int64_t memory_bytes;   /* group planning budget (plan_with_ft) */
    int workers;            /* validated >= 1; results never depend on it */
    const char* out_dir;    /* NULL/"" = temporary workspace */
    ddm_b200_before_merge_fn before_merge; /* NULL = none */
    void* before_merge_user;
    int device;             /* CUDA device ordinal */
} ddm_b200_run_config;

const char* ddm_b200_last_error(void);
int ddm_b200_version(int* major, int* minor, int* patch);
int ddm_b200_device_count(int* count);
/* Diagnostics (no reference counterpart): the kernels the last run on `device` selected, e.g.
   "spatial=rows2<256>+cols2<512> temporal=warp<1024>:map", NUL-terminated into buf. */
int ddm_b200_last_engines(int device, char* buf, int64_t capacity);

/* ddm::pad_length (proj/core/src/temporal.cpp:10-17); -1 if n < 1 */
int64_t ddm_b200_pad_length(int64_t n);
/* longest sequence the single-CTA temporal engine accepts for a precision (0 f32, 1 f64) */
int64_t ddm_b200_max_frames(int precision);

/* ddm::plan_with_ft (proj/core/src/scheduler.cpp:365-384) */
int ddm_b200_plan_with_ft(int64_t q_count, int64_t frames, int64_t bytes, int precision,
                          int64_t* capacity, int64_t* groups);

/* ddm::cutoff_set (proj/core/src/spectrum.cpp:65-84): count, and flat indices if non-NULL */
int ddm_b200_cutoff_set(int width, int height, int has_q_max, double q_max, int64_t* count,
                        int64_t* flat_out);

/* ddm::run (proj/core/src/scheduler.cpp:413-483) over an in-memory frame-major stack
   (MemoryFrameSource, frame_source.cpp:15-25).  out_values receives the lag-major f64 map,
   n_lags x height x (width/2+1) (capacity in doubles); out_lags the resolved lag list. */
int ddm_b200_run_u16(const uint16_t* pixels, int width, int height, int frames,
                     double frame_interval, const ddm_b200_run_config* config,
                     double* out_values, int64_t out_capacity, int64_t* out_lags,
                     int64_t* out_n_lags, ddm_b200_counters* counters,
                     ddm_b200_timing* timing);
/* 8-bit frames (north-star extension; values widened exactly to the u16 path's) */
int ddm_b200_run_u8(const uint8_t* pixels, int width, int height, int frames,
                    double frame_interval, const ddm_b200_run_config* config,
                    double* out_values, int64_t out_capacity, int64_t* out_lags,
                    int64_t* out_n_lags, ddm_b200_counters* counters,
                    ddm_b200_timing* timing);
/* Opaque staging session (SURVEY.md §8b "Required C-ABI"). The reference re-reads and
   re-transforms the frames on every ddm::run (scheduler.cpp:413-483); a session holds one
   stack in HBM and runs the WITH_FT branch over it for any number of wave-vector / lag
   requests. Each session owns its own device buffers and streams (its own engine, not the
   per-device one behind ddm_b200_run_*), so sessions on one GPU run concurrently; use one
   session from one thread at a time. One GPU per session: multi-GPU runs are one process per
   GPU (ddm_b200_shard_plan and the *_shard_* entries). */
typedef struct ddm_b200 ddm_b200;
/* precision 0 = f32, 1 = f64; device = CUDA ordinal */
int ddm_b200_create(int width, int height, int frames, int precision, int device, ddm_b200** out);
int ddm_b200_destroy(ddm_b200* session);
/* frames [first, first + count) of a frame-major host buffer holding exactly those frames
   (FrameSource::read_frame, frame_source.hpp:33); u16 or u8, not mixed within a session */
int ddm_b200_stage_frames(ddm_b200* session, const uint16_t* host, int first, int count);
int ddm_b200_stage_frames_u8(ddm_b200* session, const uint8_t* host, int first, int count);
/* WITH_FT over the staged stack (every frame must be staged). wv_flat: q_count ascending flat
   indices row * (width/2+1) + col (NULL = the whole half plane, q_count ignored); lags: NULL/0
   = every lag, else normalised like RunConfig::lags. out_lag_major: n_lags x height x
   (width/2+1) f64, zeros outside wv_flat, d(0) = 0 (ResultMap, result_map.hpp:12-32);
   validate() floors (archive.cpp:44-58); counters spatial_ffts = frames, temporal_ffts =
   2 q_count. A page-locked out_lag_major streams out beside the temporal pass. */
int ddm_b200_run_with_ft(ddm_b200* session, const int64_t* wv_flat, int64_t q_count,
                         const int64_t* lags, int64_t n_lags, double* out_lag_major,
                         int64_t out_capacity, ddm_b200_counters* counters,
                         ddm_b200_timing* timing);
/* the kernels the session's last run selected (like ddm_b200_last_engines) */
int ddm_b200_session_engines(ddm_b200* session, char* buf, int64_t capacity);

/* ddm::run over RawStackFileSource (frame_source.cpp:27-78) */
int ddm_b200_run_raw_stack(const char* path, const ddm_b200_run_config* config,
                           double* out_values, int64_t out_capacity, int64_t* out_lags,
                           int64_t* out_n_lags, ddm_b200_counters* counters,
                           ddm_b200_timing* timing);

/* ddm::run over PgmDirSource (frame_source.cpp:80-95): a directory of P5 / maxval 65535
   frames, sorted by file name.  Frames are read by a thread pool into pinned staging and
   streamed to HBM (as for raw stacks). */
int ddm_b200_run_pgm_dir(const char* dir, const ddm_b200_run_config* config, double* out_values,
                         int64_t out_capacity, int64_t* out_lags, int64_t* out_n_lags,
                         ddm_b200_counters* counters, ddm_b200_timing* timing);
/* `ddm analyze` (tools/ddm_cli.cpp:206-240) as one call: open the stack (format 0 raw_stack,
   1 pgm_dir, -1 auto = directory -> pgm_dir), ddm::run with the workspace in out_dir,
   write_results (d_m<lag>.bin + index.json), radial.csv (azimuthal_average +
   write_radial_csv) and, when at least 4 lags >= 1 exist, fits.csv (fit_all_bins +
   write_fits_csv).  The CLI's run.json option echo is left to the caller (the Python
   wrapper writes it).  fits_written = 1 if fits.csv was written. */
int ddm_b200_analyze(const char* path, int format, const ddm_b200_run_config* config,
                     const char* out_dir, int64_t* out_n_lags, int64_t* fits_written,
                     ddm_b200_counters* counters, ddm_b200_timing* timing);
/* `ddm bench` (tools/ddm_cli.cpp:338-385, core/src/bench.cpp): every (size, N, algorithm
   [0 with_ft, 1 without_ft, 2 direct], workers, budget) cell of a sweep over synthetic stacks
   seeded (N << 32) ^ size, run in f64 (warmup + repetitions, per-field medians), written to
   out_csv in bench.csv's format; crossover_sizes / crossover_n (capacity n_sizes) receive the
   smallest N where with_ft beats without_ft per size (-1 = none), n_crossover their count.
   Cells that fail to plan are recorded as failed rows (nan times). */
int ddm_b200_bench_sweep(const int* frame_counts, int n_frame_counts, const int* sizes, int n_sizes,
                         const int* algorithms, int n_algorithms, const int* workers, int n_workers,
                         const int64_t* budgets, int n_budgets, int repetitions, int warmup,
                         const char* out_csv, int* crossover_sizes, int* crossover_n,
                         int* n_crossover);
/* `ddm compare` (tools/ddm_cli.cpp:247-290): the stack through two algorithms (0 with_ft,
   1 without_ft, 2 direct) with `config` otherwise; deviation = max|a-b| / max(|a|,|b|),
   tolerance 1e-4 (f32) / 1e-9 (f64), pass = deviation <= tolerance.  The CLI's compare.json
   is the caller's (the Python wrapper writes it). */
int ddm_b200_compare(const char* path, int format, const ddm_b200_run_config* config, int algorithm_a,
                     int algorithm_b, double* deviation, double* tolerance, int* pass,
                     ddm_b200_timing* timing_a, ddm_b200_timing* timing_b);
/* `ddm synth` (tools/ddm_cli.cpp:306-327): generate a size x size stack (synth.cpp:98-132) and
   write out_dir/stack.raw (write_raw_stack, image_stack.cpp:223-247) and out_dir/synth.json
   (write_synth_manifest, synth.cpp:134-155). Host only. */
int ddm_b200_synth(const char* out_dir, int64_t particles, double diffusion, double psf_sigma,
                   double amplitude, double background, int size, int frames, double frame_interval,
                   uint64_t seed);
/* ddm::crossover (core/src/bench.cpp:144-183) over a table of n_cells cells (algorithm 0/1/2,
   frames, square size, median total seconds, failed flag; failed may be NULL): per size in
   first-seen order, the smallest N whose first with_ft cell beats the first without_ft cell
   (-1 = none).  sizes_out / n_star_out need room for one entry per distinct size.  Host only. */
int ddm_b200_crossover(int64_t n_cells, const int* algorithm, const int* frames, const int* width,
                       const double* seconds_total, const int* failed, int* sizes_out, int* n_star_out,
                       int* n_out);
/* Dimensions of a stack on disk (format 0 raw_stack, 1 pgm_dir; open_frame_source). */
int ddm_b200_stack_dims(const char* path, int format, int* width, int* height, int* frames);

/* ddm::load_stack (image_stack.cpp:160-247): the whole stack into out (frame-major u16,
   capacity in samples); host only. */
int ddm_b200_load_stack(const char* path, int format, uint16_t* out, int64_t capacity);

/* Device-resident WITH_FT: frames already in HBM (pixel_bytes 2 = u16, 1 = u8), map written
   to HBM as lag-major [n_lags][height*(width/2+1)] f32 (out_f64 = 0) or f64.  Positions
   outside a cutoff are left untouched.  Runs on the library's stream for `device`, ordered
   after `stream` (cudaStream_t, may be NULL) and re-joined to it on return; optional
   device times of the spatial and temporal kernels. */
int ddm_b200_run_device(const void* d_frames, int pixel_bytes, int width, int height,
                        int frames, int precision, const int64_t* lags, int64_t n_lags,
                        int has_q_max, double q_max, void* d_out, int out_f64, int device,
                        void* stream, double* spatial_ms, double* temporal_ms,
                        int* kernel_launches);

/* ---- Sharded WITH_FT over several GPUs (one process per GPU).  The reference
   runs one process; its out-of-core GroupPlan (scheduler.cpp:365-384) is what the shards
   follow, so rank r's temporal output is the PartialResult of group r (archive.hpp:48-61).
   Step 1 (spatial_shard) -> corner-turn all-to-all (NCCL, caller) -> step 2
   (temporal_segments). */

/* ddm::plan_shards: frame_begin / q_begin receive ranks + 1 offsets each. */
int ddm_b200_shard_plan(int64_t q_count, int64_t frames, int ranks, int64_t* frame_begin,
                        int64_t* q_begin);

/* Step 1 on one rank, replacing run_with_ft's frame loop (scheduler.cpp:108-127) for the
   rank's frames: d_frames [frames][height][width] (u16 / u8) -> d_spec, every wave vector of
   the half plane, q-major [height*(width/2+1)][frames] complex (f32 or f64 pairs).  The rows
   [q_begin[d], q_begin[d+1]) are the block sent to rank d. Ordered after `stream`. */
int ddm_b200_spatial_shard_device(const void* d_frames, int pixel_bytes, int width, int height,
                                  int frames, int precision, void* d_spec, int device,
                                  void* stream, double* ms);

/* Step 1 fused with the corner turn (NVLink peer stores): as spatial_shard_device, but wave
   vector k of this rank's frames is stored straight into its owner's receive buffer,
   dest[d] + (k - q_begin[d]) * frames for q_begin[d] <= k < q_begin[d+1], where dest[d] is a
   device pointer valid on this GPU (a peer mapping of rank d's buffer, already offset to this
   rank's segment).  Needs the register-resident spatial kernels (f32, power-of-two W/2 and
   H <= 1024); status 1 otherwise.  The caller orders the peers' step 2 after every rank's
   step 1 (a cross-GPU barrier). */
int ddm_b200_spatial_shard_p2p_device(const void* d_frames, int pixel_bytes, int width, int height,
                                      int frames, int precision, int ranks,
                                      const int64_t* q_begin, void* const* dest, int device,
                                      void* stream, double* ms);

/* Step 2 on one rank, replacing the per-sequence loop (scheduler.cpp:146-162) for its group:
   d_recv is the all-to-all receive buffer, [source s][q_count][seg_frames[s]] complex;
   sequence q is the concatenation of its source segments.  Writes the lag-major map
   d_out[li * out_stride + q] (f32 or f64) for the requested lags (NULL/0 = all). */
/* Sharded ring average, step 1 (SURVEY §8e "assembly"): per-(lag, ring) sums of one rank's
   wave-vector slice [q_begin, q_begin + q_count) of the plane (identity layout: no cutoff in
   the sharded run), map [n_lags][map_stride] f32 (map_f64 = 0) or f64 in HBM.  Rings are
   llround(|q|) over the whole plane (analysis.cpp:61-97; optional q_max drops wave vectors), so
   every rank returns the same bin_count; counts (host, bin_count) are the slice's ring
   populations.  d_sums NULL = size query.  Step 2 (sharded.ring_average) adds the ranks' sums
   in rank order and divides by the summed counts. */
int ddm_b200_ring_sums_device(const void* d_map, int map_f64, int64_t q_begin, int64_t q_count,
                              int64_t map_stride, int64_t n_lags, int width, int height, int has_q_max,
                              double q_max, double* d_sums, int64_t capacity, int64_t* counts,
                              int64_t* bin_count, int device, void* stream);
int ddm_b200_temporal_segments_device(const void* d_recv, int64_t q_count, int n_segments,
                                      const int64_t* seg_frames, int precision,
                                      const int64_t* lags, int64_t n_lags, void* d_out,
                                      int64_t out_stride, int out_f64, int device, void* stream,
                                      double* ms);

/* Batched SequenceEngine<S>::with_ft (proj/core/src/temporal.cpp:77-112): q sequences of n
   complex values, interleaved (re, im) f64, q-major; the working precision is `precision`
   (values are rounded to f32 first when precision = 0, as a complex<float> caller would).
   d / d_a / corr are q x n f64 (d_a and corr may be NULL), restored to the original basis. */
int ddm_b200_sequences_with_ft(const double* seq, int64_t q, int64_t n, int precision,
                               int device, double* d, double* d_a, double* corr,
                               uint64_t* temporal_ffts);

/* ddm::compute_spectra (proj/core/src/spectrum.cpp:29-63) on u16 frames: out is
   frames x height x (width/2+1) complex, interleaved f64. */
int ddm_b200_spectra_u16(const uint16_t* pixels, int width, int height, int frames,
                         int precision, int device, double* out);
/* ddm::forward_spectrum (proj/core/src/spectrum.cpp:12-27) on one real frame (f64 values). */
int ddm_b200_forward_spectrum(const double* frame, int width, int height, int precision,
                              int device, double* out);

/* ddm::azimuthal_average (proj/core/src/analysis.cpp:61-97): map is n_lags x plane f64
   (host); means n_lags x bins, counts bins; capacity = bins the caller allocated. */
int ddm_b200_azimuthal(const double* values, int64_t n_lags, int width, int height,
                       int has_q_max, double q_max, int device, double* means,
                       int64_t* counts, int64_t capacity, int64_t* bin_count);

/* ddm::run (WITH_FT) followed by ddm::azimuthal_average (analysis.cpp:61-97), the pair
   `ddm analyze` calls (tools/ddm_cli.cpp:218-225), in one device pass.  Where the register
   engines apply (f32, N2 = 2048, power-of-two frames) the ring sums are fused into the
   temporal kernel and no map is materialised (*fused = 1); otherwise the map goes through HBM
   and the ring reduction.  means: [n_lags][capacity] f64 (bins beyond bin_count zero);
   counts (optional, host): per-bin wave-vector counts; d_means = NULL queries bin_count. */
int ddm_b200_run_azimuthal_device(const void* d_frames, int pixel_bytes, int width, int height,
                                  int frames, int precision, const int64_t* lags, int64_t n_lags,
                                  int has_q_max, double q_max, double* d_means, int64_t capacity,
                                  int64_t* counts, int64_t* bin_count, int device, void* stream,
                                  double* spatial_ms, double* temporal_ms, int* fused);
/* The same over host u16 frames and a reference RunConfig; means on the host (NULL = size
   query); out_lags receives the resolved lag list. */
int ddm_b200_run_azimuthal_u16(const uint16_t* pixels, int width, int height, int frames,
                               const ddm_b200_run_config* config, double* means, int64_t capacity,
                               int64_t* counts, int64_t* bin_count, int64_t* out_lags,
                               int64_t* out_n_lags);

/* ddm::fit_all_bins / fit_exponential (analysis.cpp:108-224): d = A (1 - exp(-t / tau)) + B per
   ring, t = lag * frame_interval, over the lags >= 1 with finite means; means is the
   [n_lags][nbins] ring profile (as ddm_b200_azimuthal / run_azimuthal produce).  One warp per
   ring on the device.  Outputs are per bin (host arrays of nbins); flag 0 ok, 1 degenerate,
   2 no_converge, -1 not fitted (empty ring or fewer than 4 usable lags). */
int ddm_b200_fit_rings(const double* means, const int64_t* lags, int64_t n_lags,
                       const int64_t* counts, int64_t nbins, double frame_interval, int device,
                       double* amplitude, double* baseline, double* tau, double* residual,
                       int* flag);
/* ddm::estimate_diffusion (analysis.cpp:242-271) over the ok fits of bins [q_lo, q_hi]. */
int ddm_b200_estimate_diffusion(const double* tau, const int* flag, int64_t nbins, int64_t width,
                                int64_t q_lo, int64_t q_hi, double* coefficient,
                                int64_t* bins_used);

/* ddm::generate (proj/core/src/synth.cpp:98-132), bit-identical u16 frames. */
int ddm_b200_generate(int64_t particles, double diffusion, double psf_sigma, double amplitude,
                      double background, int width, int height, int frames,
                      double frame_interval, uint64_t seed, uint16_t* out);
/* The same frames rendered on the device into d_out ([frames][height][width] u16 in HBM):
   the generator staging frames to HBM (BASELINE north_star). Trajectories on the host with
   the reference's draw sequence; frames by a render kernel with the reference's per-pixel
   arithmetic (synth.cpp:42-79). Ordered after `stream`; returns when the frames are written. */
int ddm_b200_generate_device(int64_t particles, double diffusion, double psf_sigma,
                             double amplitude, double background, int width, int height,
                             int frames, double frame_interval, uint64_t seed, uint16_t* d_out,
                             int device, void* stream);

#ifdef __cplusplus
}
#endif

#endif
