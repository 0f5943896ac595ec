/*
 * hapi.h -- C ABI of the B200-native storage-side prefix forward of HAPI
 * (Guirguis et al., "Accelerating Transfer Learning with Near-Data Computation on
 * Cloud Object Stores", arXiv 2210.08650).  PAPER.md below = /root/reference/PAPER.md.
 *
 * The hot path: the storage side "reads the object that holds the training data and
 * the specified DNN ... and then executes the feature extraction part up to the split
 * index" and "sends back the outputs of the split index layer" (section 4.1,
 * PAPER.md:732-734), running "custom DNN models that run the forward pass between
 * arbitrary start and end layers".  The planner calls follow the
 * paper's statement of the problem: per-layer output sizes and the memory profile
 * (section 4.3), the split index (Alg. 1) and the
 * storage-side (COS) batch size under a GPU-memory budget (Eq. 4).
 *
 * Conventions (all calls):
 *   - Plain C types; pointers are host pointers unless documented as device.
 *   - Return HAPI_OK (0) or a positive hapi_status; hapi_last_error() returns a
 *     thread-local message for the last failure on the calling thread.
 *   - Layer indices s are 1-based and inclusive: s = number of leading layers run on
 *     storage (L_COS, Appendix C; reading R1).  Array slot
 *     [s-1] describes layer s.
 *   - Layers are the canonical torchvision module lists of DESIGN.md reading R2
 *     (AlexNet 21, ResNet18 14, ResNet50 22, VGG11 29, DenseNet121 22).
 */
#ifndef HAPI_H_
#define HAPI_H_

#include <stdint.h>

#if defined(__GNUC__)
#define HAPI_API __attribute__((visibility("default")))
#else
#define HAPI_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HAPI_OK = 0,
  HAPI_ERR_INVALID_ARGUMENT = 1, /* batch 0, split/freeze out of range, link 0, b_min > b_max,
                                    capacity < L, u64 overflow, null pointer */
  HAPI_ERR_INVALID_MODEL = 2,    /* unknown arch, params count/shape mismatch, image size too small */
  HAPI_ERR_INFEASIBLE = 3,       /* the HBM budget cannot hold b_min images (Eq. 4 has no solution;
                                    the single-request analog of "removes one request ... and
                                    retries") */
  HAPI_ERR_OUT_OF_MEMORY = 4,    /* device allocation failed */
  HAPI_ERR_CUDA = 5,             /* a CUDA runtime/driver call failed (incl. earlier async faults) */
  HAPI_ERR_UNSUPPORTED = 6       /* valid request this build does not implement */
} hapi_status;

typedef enum { HAPI_ALEXNET = 0, HAPI_RESNET18 = 1, HAPI_RESNET50 = 2, HAPI_VGG11 = 3,
               HAPI_DENSENET121 = 4 } hapi_arch;

/* Activation dtype of the prefix.  F32: fp32 activations, fp32 SIMT math (the paper's
 * precision, reading R7).  BF16: bf16 activations, fp32 accumulation on tcgen05 tensor
 * cores.  Images are always fp32 NCHW. */
typedef enum { HAPI_F32 = 0, HAPI_BF16 = 1 } hapi_dtype;

/* ------------------------------------------------------------------ planner (host) */

/* Number of canonical layers L of `arch`, or -HAPI_ERR_INVALID_MODEL. Pure. */
HAPI_API int32_t hapi_num_layers(hapi_arch arch);

/* Table 2 freeze index of `arch`, or -HAPI_ERR_INVALID_MODEL. Pure. */
HAPI_API int32_t hapi_freeze_index(hapi_arch arch);

/* Per-layer facts for s = 1..L (slot s-1); Alg. 1 profile_model
 * computed analytically (shapes are static, so no profiling run is needed):
 *   input_bytes  l0 = 3*in_h*in_w*4   (the fp32 input sample, Alg. 1 line 9; reading A3)
 *   out_bytes    l_s = numel(output of layer s) * sizeof(act)
 *   peak_bytes   P(s) = max_{1<=i<=s} (l_{i-1} + l_i)   ("maximum input plus output size
 *                across all layers", section 4.3)
 *   weight_bytes W(s) = sum_{i<=s} weight elems*sizeof(act) + (bias + BN gamma,beta elems)*4
 * Any output pointer may be NULL.  capacity = length of the caller's arrays (>= L).
 * Pure, re-entrant, no device work.  Errors: INVALID_MODEL (arch, or an empty layer
 * output at this image size), INVALID_ARGUMENT (capacity < L, overflow). */
HAPI_API hapi_status hapi_layer_sizes(hapi_arch arch, uint32_t in_h, uint32_t in_w, hapi_dtype act,
                             uint64_t *input_bytes, uint64_t *out_bytes, uint64_t *peak_bytes,
                             uint64_t *weight_bytes, uint32_t capacity);

typedef struct {
  hapi_arch arch;
  uint32_t in_h, in_w;        /* image size (224 x 224 for ImageNet, reading R6) */
  hapi_dtype act;             /* sizes are counted in this dtype */
  uint32_t freeze_idx;        /* 1..L; Table 2 defaults 17, 11, 21, 25, 20 */
  uint64_t training_batch;    /* >= 1 */
  uint64_t link_bytes_per_s;  /* > 0; 1 Gbps = 125,000,000 B/s (reading A4) */
  uint32_t threshold_ms;      /* >= 1; 1000 = "network bandwidth times 1s" */
  uint64_t hbm_budget_bytes;  /* memory the storage side may use on this GPU
                                 (M_total - M_occupied of Eq. 4) */
  uint32_t b_min, b_max;      /* COS batch bounds: b_min = 25; b_max <= training
                                 batch. 1 <= b_min <= b_max */
} hapi_split_query;

typedef struct {
  uint32_t split_idx;           /* Alg. 1 winner in 1..freeze_idx */
  uint32_t cos_batch;           /* min(b_max, floor((budget - W(s)) / P(s))); 0 if infeasible */
  uint64_t bytes_per_iteration; /* l_split * training_batch */
  uint64_t est_bytes;           /* W(s) + cos_batch * P(s) */
  uint32_t n_candidates;        /* |{l <= freeze : l_l < l0}| */
} hapi_split_result;

/* Alg. 1 choose_split_idx + Eq. 4 for one request:
 *   candidates = {l <= freeze : l_l < l0} ascending; C = link_bytes_per_s*threshold_ms/1000;
 *   split = first candidate with l_l * training_batch < C, else freeze_idx (both
 *   comparisons strict, reading A5; line 16 read as `winner = l`, reading A6);
 *   cos_batch = largest b in [b_min, b_max] with W(s) + b*P(s) <= budget.
 * `candidates` (optional, may be NULL) receives n_candidates indices; it must hold L.
 * Returns HAPI_ERR_INFEASIBLE with r fully filled (cos_batch = 0, est = W(s)) when b_min
 * does not fit.  All arithmetic u64 with overflow -> INVALID_ARGUMENT.  Pure. */
HAPI_API hapi_status hapi_choose_split(const hapi_split_query *q, hapi_split_result *r, uint32_t *candidates);

/* ------------------------------------------------------------ batch adaptation (host)
 * Section 4.5: the COS batch of every queued
 * request of one GPU from Eq. 4,
 *     max sum_r b_r*M_r(data) + M_r(model)
 *     s.t. b_min,r <= b_r <= b_max,r,   sum_r b_r*M_r(data) + M_r(model) <= available_bytes,
 * with M_r(model) = W(s_r) and M_r(data) = P(s_r) from hapi_layer_sizes, and
 * available_bytes = M_total - M(occupied).  The paper states the problem, not a solver;
 * readings:
 *   F1 infeasible -> requests are removed one at a time, most recent arrival first
 *      ("removes one request at a time and retries"); they get batch 0
 *      (deferred to the next run), so the deferred set is a suffix of arrival order;
 *   F2 solver = unit water-filling: every kept request starts at b_min, then one more sample
 *      goes to the request with the smallest current b (earliest arrival on ties) that is below
 *      b_max and whose M(data) still fits, until none does -- the objective is within
 *      max_r M_r(data) of the optimum;
 *   F3 max_concurrency > 0 (the static cap) defers every request beyond the
 *      first max_concurrency by arrival; 0 = no cap;
 *   F4 hapi_partition_requests spreads requests (in arrival order) round-robin over GPUs
 *      ("distributes requests evenly on the existing GPUs").
 * Pure, deterministic, no device work. */
typedef struct {
  uint64_t arrival_seq;           /* arrival order key (ties: input order) */
  uint64_t model_bytes;           /* M_r(model) */
  uint64_t data_bytes;            /* M_r(data) per sample */
  uint32_t b_min, b_max;          /* 1 <= b_min <= b_max (b_min = 25 in the paper) */
} hapi_adapt_request;

/* batch[i] <- b_i (0 = deferred) for the n requests in input order; *used_bytes (may be NULL)
 * <- memory of the kept requests.  Errors: INVALID_ARGUMENT (null arrays with n > 0, bad
 * bounds).  n = 0 is valid (nothing assigned, 0 bytes). */
HAPI_API hapi_status hapi_adapt_batches(const hapi_adapt_request *reqs, uint32_t n, uint64_t available_bytes,
                                        uint32_t max_concurrency, uint32_t *batch, uint64_t *used_bytes);

/* gpu_of[i] <- GPU of the i-th request in arrival order (round-robin, F4).  Errors:
 * INVALID_ARGUMENT (n_gpus = 0, null gpu_of with n > 0). */
HAPI_API hapi_status hapi_partition_requests(uint32_t n, uint32_t n_gpus, uint32_t *gpu_of);

/* ------------------------------------------------------------------ server loop (f1)
 * The batch-adaptation loop of one GPU (section 4.5): requests are
 * queued; a round of hapi_adapt_batches runs "when two conditions hold: (1) there is
 * available GPU memory for new requests, and (2) there exists at least one queued request
 * that has not yet been accounted for in the previous runs", after the server "waits for
 * new requests for a small amount of time"; requests the round cannot fit "become part of
 * the next batch assignment round, typically after some existing requests finish".
 * Readings:
 *   F5 the round runs at the first poll with now >= (earliest unaccounted arrival) + wait_us;
 *   F6 available = total - occupied - sum over running requests of (W_r + b_r * P_r);
 *      condition (1) = available > 0 and (no cap, or fewer running requests than the cap);
 *   F7 a round considers the unaccounted and the deferred requests, with the static cap
 *      reduced by the running count; admitted requests run, the others become deferred;
 *   F8 hapi_scheduler_finish returns the request's memory and makes deferred requests
 *      unaccounted again (original arrival times kept).
 * Host-only, deterministic (the caller supplies the clock), not thread-safe per handle. */
typedef struct hapi_scheduler hapi_scheduler;
typedef enum { HAPI_REQ_QUEUED = 0, HAPI_REQ_DEFERRED = 1, HAPI_REQ_RUNNING = 2, HAPI_REQ_DONE = 3 } hapi_req_state;
typedef struct {
  uint64_t total_bytes;           /* M_total of the GPU */
  uint64_t occupied_bytes;        /* M(occupied): CUDA/framework reservation estimated by the provider */
  uint32_t max_concurrency;       /* static cap on running requests; 0 = none */
  uint64_t wait_us;               /* the wait window (F5) */
} hapi_scheduler_config;
/* Errors: INVALID_ARGUMENT (null, occupied > total). */
HAPI_API hapi_status hapi_scheduler_create(const hapi_scheduler_config *cfg, hapi_scheduler **out);
/* Queue a request arriving at now_us (non-decreasing across calls): r->arrival_seq is ignored
 * (arrival = now_us, ties by submission order); *id <- its handle (0, 1, 2, ...).
 * Errors: INVALID_ARGUMENT (null, bad bounds, now_us earlier than a previous call). */
HAPI_API hapi_status hapi_scheduler_submit(hapi_scheduler *s, uint64_t now_us, const hapi_adapt_request *r,
                                           uint64_t *id);
/* Run a round if the trigger holds at now_us: ids[k], batches[k] <- the admitted requests in
 * arrival order (k < *n_admitted <= cap; a round admitting more than cap is an
 * INVALID_ARGUMENT before any state change).  *n_admitted = 0 when no round ran. */
HAPI_API hapi_status hapi_scheduler_poll(hapi_scheduler *s, uint64_t now_us, uint64_t *ids, uint32_t *batches,
                                         uint32_t cap, uint32_t *n_admitted);
/* A running request completed.  Errors: INVALID_ARGUMENT (unknown id, not running). */
HAPI_API hapi_status hapi_scheduler_finish(hapi_scheduler *s, uint64_t id);
/* State and COS batch (0 unless running) of request id; *available <- F6 available bytes. */
HAPI_API hapi_status hapi_scheduler_query(const hapi_scheduler *s, uint64_t id, uint32_t *state, uint32_t *batch,
                                          uint64_t *available);
HAPI_API void hapi_scheduler_destroy(hapi_scheduler *s);

/* Parameters expected by hapi_model_create, in torchvision state_dict order
 * (num_batches_tracked buffers excluded): count, and per index the name (copied into
 * name_buf, NUL-terminated, truncated to name_cap) and shape (dims[4], *ndim). */
HAPI_API int32_t hapi_num_params(hapi_arch arch);
HAPI_API hapi_status hapi_param_info(hapi_arch arch, uint32_t idx, char *name_buf, uint32_t name_cap,
                            int64_t dims[4], uint32_t *ndim);

/* ------------------------------------------------------------------ executor (device) */
/* (the model API is below; the serving loop that drives it, hapi_server, follows it) */

typedef struct hapi_model hapi_model;

typedef struct {
  hapi_arch arch;
  hapi_dtype act;
  uint32_t in_h, in_w;       /* image size; 224 x 224 for every config (reading R6) */
  uint32_t min_split, max_split; /* plans are prepared for split_idx in [min_split, max_split],
                                    1 <= min <= max <= L; weights of layers 1..max_split are
                                    kept on the device */
  uint32_t max_batch;        /* arena sized for this many images per launch (normally the
                                 cos_batch of hapi_choose_split); larger calls are chunked */
  int device;                /* CUDA ordinal.  Every call on the model switches to it and
                                 restores the caller's current device on return. */
  uint32_t host_chunk;       /* images per chunk of hapi_prefix_forward_host (0: no host
                                path).  Its staging -- 2 x host_chunk images in and split
                                outputs out, the double-buffered DRAM<->GPU transfers of
                                Eq. 1's C11 * B * (l0 + l_split) terms, PAPER.md:204-206 --
                                is allocated here at create time and counted in
                                hapi_model_device_bytes; min(host_chunk, max_batch) is used */
} hapi_model_desc;

/* Builds a model: reads the fp32 host params (read during the call only; caller keeps
 * ownership), folds eval-mode BatchNorm into the preceding conv in fp64 where the plan
 * allows it, converts/packs weights for the kernels, uploads them, allocates the arena
 * and builds one launch plan per split.  Errors: INVALID_ARGUMENT (desc), INVALID_MODEL
 * (n_params != hapi_num_params, unsupported image size), OUT_OF_MEMORY, CUDA. */
HAPI_API hapi_status hapi_model_create(const hapi_model_desc *desc, const float *const *params,
                              uint32_t n_params, hapi_model **m);

/* A model over the SAME device weights as `base` (no copy; the weights are freed with the
 * last model that holds them), with its own plans, arena for max_batch images and host
 * staging (host_chunk, 0 = none): concurrent requests of one (arch, split range) share one
 * copy of the frozen weights (f1).  Its hapi_model_device_bytes reports 0 weight bytes (they
 * are counted once, on the base).  Errors: INVALID_ARGUMENT, OUT_OF_MEMORY, CUDA. */
HAPI_API hapi_status hapi_model_create_shared(const hapi_model *base, uint32_t max_batch, uint32_t host_chunk,
                                              hapi_model **out);

/* Stream for subsequent launches (a cudaStream_t; NULL = legacy default stream). */
HAPI_API hapi_status hapi_model_set_stream(hapi_model *m, void *cuda_stream);

/* The hot path.  images: DEVICE pointer, [batch,3,in_h,in_w] fp32 NCHW contiguous.
 * out: DEVICE pointer with room for batch * out_bytes[split_idx-1] bytes; receives the
 * layer-split_idx activations as contiguous NCHW [batch,C,H,W] (or [batch,F] inside a
 * classifier) in the model's act dtype (reading R11).  Images are processed in chunks
 * of max_batch in order; results do not depend on chunking (a8).  Asynchronous on the
 * model's stream; never allocates device memory (the first call per (split, chunk size)
 * captures and instantiates a CUDA graph; later calls with other buffers update it in
 * place).  images/out must not alias each other or the model.
 * Errors: INVALID_ARGUMENT (batch 0, split outside [min_split,max_split], null),
 * CUDA (launch failure or an earlier asynchronous fault). */
HAPI_API hapi_status hapi_prefix_forward(hapi_model *m, uint32_t split_idx, const float *images,
                                uint64_t batch, void *out);

/* Client-side frozen suffix ("the client ... runs the
 * remaining layers", PAPER.md:902-906 frozen layers up to the freeze index): a model whose
 * input is layer `start_idx`'s output in the send-buffer layout (contiguous NCHW, act dtype,
 * exactly what hapi_prefix_forward writes at split = start_idx) and which computes layers
 * start_idx+1 .. end_idx for end_idx in [min_split, max_split].  Same kernels and fusions as
 * the prefix; weights of layers <= start_idx are never read.  Requires
 * 1 <= start_idx < min_split; everything else as hapi_model_create.  Such a model only
 * accepts hapi_suffix_forward (the prefix entry points return INVALID_ARGUMENT). */
HAPI_API hapi_status hapi_model_create_suffix(const hapi_model_desc *desc, uint32_t start_idx,
                                              const float *const *params, uint32_t n_params, hapi_model **out);

/* acts: device [batch, layer start_idx output] (act dtype, contiguous NCHW); out: device,
 * batch * l_end bytes, contiguous NCHW of layer end_idx.  Chunked by max_batch like the
 * prefix.  Errors: INVALID_ARGUMENT (not a suffix model, end_idx out of range, null, batch 0),
 * CUDA. */
HAPI_API hapi_status hapi_suffix_forward(hapi_model *m, uint32_t end_idx, const void *acts, uint64_t batch,
                                         void *out);

/* End-to-end variant with HOST buffers (pinned or pageable): images [batch,3,H,W] fp32
 * host -> device copies, prefix forward, device -> host copy of the split output into
 * host `out`, pipelined in chunks of at most desc.host_chunk images (a half-size first
 * chunk: its H2D is the pipeline fill) over two copy streams (H2D of chunk i+1 and D2H of
 * chunk i-1 overlap compute of chunk i; "moving data to and from GPU").
 * Uses only the staging allocated at create time (never allocates).  Synchronous:
 * returns when `out` is filled.  Errors: INVALID_ARGUMENT (host_chunk was 0, batch 0,
 * split out of range, null), CUDA. */
HAPI_API hapi_status hapi_prefix_forward_host(hapi_model *m, uint32_t split_idx, const float *images,
                                     uint64_t batch, void *out);

/* The same, enqueued without waiting: returns once the copies and launches are queued.
 * Calls may follow each other back to back -- the staging slots alternate across calls, so
 * the H2D of the next call overlaps the compute of the previous one (a stream of requests
 * pays the pipeline fill and drain once).  `images` must stay valid and `out` unread until
 * hapi_host_sync(m) returns.  Errors as hapi_prefix_forward_host. */
HAPI_API hapi_status hapi_prefix_forward_host_async(hapi_model *m, uint32_t split_idx, const float *images,
                                                   uint64_t batch, void *out);
/* Wait for every host-path call enqueued on the model (its copy streams and its stream). */
HAPI_API hapi_status hapi_host_sync(hapi_model *m);

/* u8 ingest (optional): images arrive as uint8 NCHW [batch,3,in_h,in_w]
 * (what an image decoder produces; a quarter of the fp32 PCIe bytes of the host path, the
 * "moving data to and from GPU" overhead of PAPER.md:911) and the input pack kernel turns each
 * value u of channel c into scale[c] * u + shift[c] in fp32 before the same packing -- the
 * caller's normalisation (e.g. scale = 1/(255 std), shift = -mean/std) folded into the ingest.
 * Everything downstream is the fp32 path's (same plans, kernels and fusions).
 * hapi_model_set_u8_norm: the per-channel scale[3] / shift[3] (host arrays, finite; default
 * scale 1/255, shift 0); waits for the model's stream, drops the u8 graphs it captured.
 * hapi_prefix_forward_u8: device images, otherwise as hapi_prefix_forward.
 * hapi_prefix_forward_host_u8 / _host_async_u8: host images, otherwise as the fp32 host calls.
 * Errors as the fp32 calls; INVALID_ARGUMENT for a suffix model. */
HAPI_API hapi_status hapi_model_set_u8_norm(hapi_model *m, const float *scale, const float *shift);
HAPI_API hapi_status hapi_prefix_forward_u8(hapi_model *m, uint32_t split_idx, const uint8_t *images,
                                            uint64_t batch, void *out);
HAPI_API hapi_status hapi_prefix_forward_host_u8(hapi_model *m, uint32_t split_idx, const uint8_t *images,
                                                 uint64_t batch, void *out);
HAPI_API hapi_status hapi_prefix_forward_host_async_u8(hapi_model *m, uint32_t split_idx, const uint8_t *images,
                                                       uint64_t batch, void *out);

/* Device bytes owned by the model: packed weights (+bias/BN vectors), and the activation
 * arena plus the host-path staging (desc.host_chunk) in *arena_bytes. */
HAPI_API hapi_status hapi_model_device_bytes(const hapi_model *m, uint64_t *weight_bytes, uint64_t *arena_bytes);

/* Per-launch profile of split_idx's plan (for bench.py's roofline): number of kernel
 * launches per chunk, and for launch i (< cap): a kernel-class id (0 conv_tc, 1 conv_simt,
 * 2 pool, 3 pack, 4 eltwise), algorithmic FLOPs and algorithmic bytes per image. */
HAPI_API hapi_status hapi_plan_info(const hapi_model *m, uint32_t split_idx, uint32_t *n_launches,
                           uint32_t *kind, double *flops_per_img, double *bytes_per_img,
                           uint32_t cap);

/* Human-readable description of launch `op` of split_idx's plan (kernel, shape, fusions),
 * NUL-terminated into buf[cap].  Diagnostics only. */
HAPI_API hapi_status hapi_plan_describe(const hapi_model *m, uint32_t split_idx, uint32_t op, char *buf, uint32_t cap);

/* Same as hapi_prefix_forward on one chunk (batch <= max_batch), recording a CUDA event
 * before and after every launch; per-launch milliseconds are written to ms[i] (< cap)
 * after an internal stream synchronize.  Instrumentation for measurement only. */
HAPI_API hapi_status hapi_prefix_forward_timed(hapi_model *m, uint32_t split_idx, const float *images,
                                      uint64_t batch, void *out, float *ms, uint32_t cap);

HAPI_API void hapi_model_destroy(hapi_model *m);

/* ------------------------------------------------------------------ serving loop (f1, device)
 * The HAPI server of one GPU (section 4.5): frozen models are registered
 * once (their weights shared by every request), requests are queued with their device
 * images and output buffers, and each hapi_server_step (1) retires requests whose forward
 * has completed (hapi_scheduler_finish), (2) runs the scheduler (trigger, wait window,
 * Eq. 4 round) and (3) launches every admitted request on its own stream: a model sharing
 * the registered weights with an arena for its COS batch b_r, hapi_prefix_forward over the
 * request's images in chunks of b_r.  Eq. 4 sizes per request are W(s), P(s) of
 * hapi_layer_sizes (M_r(model), M_r(data)); b_max is the request's (the client's training
 * batch) and b_min the provider's (25 in the paper; clipped to
 * b_max).  Not thread-safe per handle. */
typedef struct hapi_server hapi_server;
typedef struct {
  hapi_scheduler_config sched;    /* memory model, static cap, wait window */
  int device;                     /* CUDA ordinal */
  uint32_t b_min;                 /* provider's minimum COS batch */
} hapi_server_config;
HAPI_API hapi_status hapi_server_create(const hapi_server_config *cfg, hapi_server **out);
/* Register a frozen model (desc->max_batch, host_chunk are ignored); *model_id <- its handle.
 * Requests may use any split in [desc->min_split, desc->max_split]. */
HAPI_API hapi_status hapi_server_add_model(hapi_server *s, const hapi_model_desc *desc, const float *const *params,
                                           uint32_t n_params, uint32_t *model_id);
/* Queue a request at now_us: `n` device images [n,3,H,W] fp32 -> device `out` (n * l_split
 * bytes, contiguous NCHW, as hapi_prefix_forward); both owned by the caller and untouched
 * until the request is DONE.  *req_id <- its handle. */
HAPI_API hapi_status hapi_server_submit(hapi_server *s, uint64_t now_us, uint32_t model_id, uint32_t split_idx,
                                        uint32_t b_max, const float *images, uint64_t n, void *out,
                                        uint64_t *req_id);
/* One iteration of the loop at now_us (see above).  *n_active <- requests not yet DONE. */
HAPI_API hapi_status hapi_server_step(hapi_server *s, uint64_t now_us, uint32_t *n_active);
/* State (hapi_req_state) and COS batch of a request; *device_bytes (may be NULL) <- bytes the
 * server holds on the device right now (registered weights + running requests' arenas). */
HAPI_API hapi_status hapi_server_query(const hapi_server *s, uint64_t req_id, uint32_t *state, uint32_t *batch,
                                       uint64_t *device_bytes);
/* Waits for running requests, then frees everything. */
HAPI_API void hapi_server_destroy(hapi_server *s);

/* Thread-local message describing the last error on this thread ("" if none). */
HAPI_API const char *hapi_last_error(void);

/* Build identification string (compile target, version). */
HAPI_API const char *hapi_build_info(void);

#ifdef __cplusplus
}
#endif

#endif /* HAPI_H_ */
