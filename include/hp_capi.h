/*
 * hp_capi.h — the C-ABI boundary of the B200 adaptive-bitwidth linear path.
 *
 * Everything the reference's planning interfaces (proj/include/hetplan/…)
 * need from the GPU goes through these entry points: plain pointers and
 * sizes, no C++ or torch types, no exceptions across the ABI, reentrant,
 * stream-ordered. Status codes mirror the reference CLI's exit codes
 * (/root/reference/proj/tools/hetplan_main.cpp:39-42): 0 ok, 2 invalid
 * input, 3 infeasible, 4 time-limit; CUDA/NCCL failures get their own codes.
 * The C++ wrappers in include/hetplan/{quant,qlinear,plan,runtime} rethrow
 * them as the reference's exception types (std::invalid_argument,
 * hetplan::infeasible_error, std::runtime_error).
 *
 * All device pointers are caller-owned. There is no CPU fallback: on a box
 * without a usable sm_100 device every compute entry point returns HP_ECUDA.
 *
 * Which reference interface each entry point replaces is noted per function
 * (the reference has no GPU code at all — /root/reference/SPEC.md:8 — so
 * "replaces" means: the CPU function whose semantics the kernel reproduces).
 */
#ifndef HP_CAPI_H
#define HP_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HP_OK = 0,
    HP_EINTERNAL = 1,
    HP_EINVAL = 2,       /* reference exit code 2 (std::invalid_argument) */
    HP_EINFEASIBLE = 3,  /* reference exit code 3 (infeasible_error)      */
    HP_ETIMEOUT = 4,     /* reference exit code 4 (time-limited incumbent)*/
    HP_ECUDA = 5,
    HP_ENCCL = 6
} hp_status;

/* Opaque CUDA stream (cudaStream_t); NULL = legacy default stream. */
typedef void* hp_stream;

/* Thread-local message of the last failing call on this thread. */
const char* hp_last_error(void);
/* ABI version; bumped on any layout or signature change. */
int hp_abi_version(void);
/* 1 if a CUDA device with compute capability 10.x is usable, else 0. */
int hp_device_ok(void);
/* Cap the persistent K3/K4 grid at `sms` CTAs (0 = every SM), leaving SMs
 * to NCCL kernels that run concurrently in pipeline mode.               */
void hp_set_sm_budget(int sms);
/* Programmatic dependent launch between consecutive K3/K4/glue kernels on a
 * stream (default on): the next kernel's prologue and weight streaming
 * overlap the previous kernel's tail; its activation reads wait.        */
void hp_set_pdl(int enable);

/* Quantizer scheme / rounding — numeric values match the order of
 * hetplan::indicator::quant_scheme / rounding_mode (indicator.hpp:22-23). */
enum { HP_ASYMMETRIC = 0, HP_SYMMETRIC = 1 };
enum { HP_NEAREST = 0, HP_STOCHASTIC = 1 };
/* Execution phase (hetplan::memcost::phase, memcost.hpp:14). */
enum { HP_PREFILL = 0, HP_DECODE = 1 };
/* Fused epilogue flags for hp_qlinear. */
enum { HP_EPI_NONE = 0, HP_EPI_RELU = 1 };

/* ---- packed weight format ------------------------------------------------
 * W is [n_out × k_in] bf16 row-major (y = x · Wᵀ). Groups of HP_GROUP
 * consecutive elements along k_in share one step (scale) and zero.
 * Tiles of 128 rows × 128 k are stored contiguously; see DESIGN.md §3 for
 * the bit layout. For n_out % 128 == 0 and k_in % 128 == 0 the packed
 * buffer is exactly ceil(n_out·k_in·bits/8) bytes — the packed-size contract
 * of memcost::decoder_weight_bytes (memcost.cpp:15-18,30-36). Scales and
 * zeros are fp32, one per (row, group), stored tile-major as well.       */
#define HP_GROUP 128

typedef struct {
    int64_t n_out;
    int64_t k_in;
    int32_t bits;    /* 3, 4, 8 or 16 (16 = bf16 passthrough)           */
    int32_t scheme;  /* HP_ASYMMETRIC / HP_SYMMETRIC                     */
    const void* packed; /* hp_packed_bytes() bytes                       */
    const float* scale; /* hp_scale_count() floats (NULL when bits==16)  */
    const float* zero;  /* hp_scale_count() floats, asymmetric only      */
} hp_qweight;

int64_t hp_packed_bytes(int64_t n_out, int64_t k_in, int bits);
int64_t hp_scale_count(int64_t n_out, int64_t k_in);

/* K1 — group-wise quantize + pack (bit-exact with the reference quantizer
 * applied per group: /root/reference/proj/src/indicator.cpp:19-56 with
 * scaling_factor :82-91; round-to-nearest only, ties half-up).
 *   w       device bf16 [n_out × ldw], ldw ≥ k_in
 *   packed  device, hp_packed_bytes()      scale/zero device, hp_scale_count()
 *   step64/zero64  optional device fp64 [n_out × ceil(k_in/128)] row-major,
 *           the reference's step and grid origin per group (for parity).
 * bits == 16 stores bf16 verbatim in tile order (reference: quantize() is the
 * identity at 16, indicator.cpp:21).                                       */
hp_status hp_quant_pack(const void* w, int64_t n_out, int64_t k_in,
                        int64_t ldw, int bits, int scheme, int rounding,
                        void* packed, float* scale, float* zero,
                        double* step64, double* zero64, hp_stream stream);

/* K1 with K2's weight reduction fused: hp_quant_pack,
 * plus the op's indicator weight statistics from the same pass over W:
 * stats5[0] = d_w = n_out·k_in, [1] = w_min, [2] = w_max (exact; the
 * layout of hp_indicator_stats). stats5 is a DEVICE pointer (5 doubles);
 * [3..4] are not touched — hp_indicator_stats(w = NULL, x, ...) fills
 * them without re-reading W.                                               */
hp_status hp_quant_pack_stats(const void* w, int64_t n_out, int64_t k_in,
                              int64_t ldw, int bits, int scheme, int rounding,
                              void* packed, float* scale, float* zero,
                              double* step64, double* zero64, double* stats5,
                              hp_stream stream);

/* Unpack (parity/inspection): stored codes as u8 [n_out × k_in] row-major
 * (symmetric codes carry the +hi offset, hi = 2^(bits-1)-1), and fp32
 * scale/zero [n_out × groups] row-major. For bits==16, `codes` receives the
 * bf16 words (2 bytes per element). Any output may be NULL.             */
hp_status hp_quant_unpack(const hp_qweight* w, void* codes, float* scale_rm,
                          float* zero_rm, hp_stream stream);

/* Dequantize to bf16 [n_out × k_in]: zero + code·step rounded to bf16
 * (reference dequant formula indicator.cpp:53; the GEMM kernels use the
 * same per-element arithmetic).                                          */
hp_status hp_dequant(const hp_qweight* w, void* w_bf16, hp_stream stream);

/* K2 — quantization-variance indicator statistics for one operator
 * (hetplan::indicator::operator_stats, indicator.hpp:31-38):
 *   stats5[0] = d_w = n_out·k_in, [1] = w_min, [2] = w_max (exact),
 *   [3] = x_mean, [4] = x_var (population, fp64 accumulation) over all
 *   tokens·k_in elements of the calibration input x [tokens × ldx] bf16.
 * stats5 is a DEVICE pointer (5 doubles). x may be NULL (x stats = 0).
 * w may be NULL (then n_out/ldw are ignored and stats5[0..2] are left as
 * they are: the weight part of hp_quant_pack_stats).                     */
hp_status hp_indicator_stats(const void* w, int64_t n_out, int64_t k_in,
                             int64_t ldw, const void* x, int64_t tokens,
                             int64_t ldx, double* stats5, hp_stream stream);

/* K3 / K4 — y[m × n_out] = epi(x[m × k_in] · dequant(W)ᵀ) (+ residual).
 *   x   device bf16, row stride ldx elements (ldx % 8 == 0)
 *   y   device bf16, row stride ldy;  residual (nullable) stride ldr
 *   phase HP_DECODE selects the skinny-M (M = ξ) schedule with split-K,
 *   HP_PREFILL the wide-M tile schedule. Both run tcgen05 MMAs with the
 *   dequantized weights in tensor memory.
 *   workspace: hp_qlinear_workspace_bytes() bytes of device memory (may be
 *   NULL when that is 0), zero-initialised once by the caller; kernels
 *   leave it zeroed again on exit.                                         */
size_t hp_qlinear_workspace_bytes(const hp_qweight* w, int64_t m, int phase);
hp_status hp_qlinear(const hp_qweight* w, const void* x, int64_t ldx,
                     int64_t m, void* y, int64_t ldy, const void* residual,
                     int64_t ldr, int epilogue, int phase, void* workspace,
                     size_t workspace_bytes, hp_stream stream);

/* Glue (decoder-layer LayerNorm, glue.cu): y[r] = LN(x[r])*gamma + beta for
 * r < rows, fp32 statistics, eps 1e-5; h % 8 == 0, 16-byte aligned rows.  */
hp_status hp_layernorm(const void* x, int64_t ldx, int64_t rows, int64_t h, const void* gamma,
                       const void* beta, void* y, int64_t ldy, hp_stream stream);

/* Decoder glue (decoder.cu), device pointers, bf16
 * unless noted. qkv rows are [q | k | v] (h columns each, head hd-column
 * blocks); hd = 64 or 128. The K/V cache of a layer is head-major
 * [B][h/hd][S_max][hd] for K and for V (the 2*v*(s+n)*h1 elements of
 * memcost.cpp:38-42; one (request, head) context is contiguous).
 *  hp_embed: x[r] = E[tok[r]] + P[pos(r) + 2] (OPT learned positions;
 *    pos(r) = pos0 + r % s_tokens if pos_per_req else pos0; P may be NULL).
 *  hp_attention_prefill: causal self-attention of `reqs` requests of s
 *    tokens (rows r*s..), writing their K/V rows 0..s-1 into the cache at
 *    requests req0.. ; out [reqs*s x h].
 *  hp_attention_decode: one query row per request (rows = requests
 *    req0..), appends K/V at position p, attends over cache rows 0..p;
 *    split > 1 cuts the context into `split` CTAs per (request, head) whose
 *    partials merge deterministically (workspace of
 *    hp_attention_decode_workspace_bytes, zeroed once, self-resetting).
 *  hp_argmax: tok[r] = argmax_v logits[r][v] (ties -> lowest id), int32.  */
hp_status hp_embed(const int32_t* tok, int rows, int pos0, int pos_per_req, int s_tokens,
                   const void* E, const void* P, int64_t pos_s, int64_t h, int64_t vocab, void* x,
                   hp_stream stream);
hp_status hp_attention_prefill(const void* qkv, int reqs, int s, int64_t h, int hd, void* out,
                               void* k_cache, void* v_cache, int req0, int s_max, hp_stream stream);
size_t hp_attention_decode_workspace_bytes(int rows, int64_t h, int hd, int split);
hp_status hp_attention_decode(const void* qkv, int rows, int64_t h, int hd, int p, void* out,
                              void* k_cache, void* v_cache, int req0, int s_max, int split,
                              void* workspace, size_t ws_bytes, hp_stream stream);
hp_status hp_argmax(const void* logits, int64_t ld, int rows, int64_t vocab, int32_t* tok,
                    hp_stream stream);

/* ---- pipeline executor (one process per GPU, NCCL P2P at boundaries) ----
 * plan_json: a plan document (schema of hetplan_main.cpp:190-224, loaded by
 * hetplan::plan_io); stage `rank` of the plan runs on this process's current
 * CUDA device. model_json: the config "model" section ({"preset": ...} or
 * explicit fields, config.cpp:55-69). nccl_ids: `world` ncclUniqueIds of
 * 128 bytes (id l names the link rank l -> (l+1) % world), produced by
 * hp_nccl_unique_id on rank 0 and broadcast by the caller; NULL if world==1.
 * The unit order follows pipesim::make_schedule / simulate semantics
 * (/root/reference/proj/src/pipesim.cpp:22-248).                          */
typedef struct hp_pipeline hp_pipeline;
typedef struct {
    int32_t scheme;      /* HP_SYMMETRIC (default) / HP_ASYMMETRIC         */
    int32_t use_graphs;  /* capture the round into one CUDA graph          */
    int32_t instrument;  /* CUDA events around the linear ops of 1 unit/phase */
    int32_t sm_budget;   /* persistent-kernel grid cap, 0 = all SMs         */
    uint64_t seed;       /* synthetic tensors (oracle/synth.py mirror)     */
    double weight_std;   /* synthetic weight std (0.02)                    */
    double timeout_s;    /* hp_pipeline_run watchdog, 0 = none; expiry ->
                          * HP_ETIMEOUT with per-stream progress in
                          * hp_last_error (destroy the pipeline after)     */
} hp_pipeline_options;
/* Weight loader sources (the paper's on-the-fly quantized loader,
 * PAPER.md:806-811, 827-828): each bf16 tensor comes from host memory
 * (pinned: copied directly; pageable: staged through pinned bins) or a raw
 * little-endian bf16 file at a byte offset; {NULL, NULL, 0} = the seeded
 * synthetic tensor. Tensors stream to the device in bins of bin_bytes
 * (0 -> 64 MiB) and K1 packs bin i while bin i+1 is copied.             */
typedef struct {
    const void* host;
    const char* path;
    int64_t offset;
} hp_tensor_src;
typedef struct {
    int32_t n_layers;            /* the plan's num_layers                       */
    const hp_tensor_src* linear; /* [n_layers*4] qkv [3h1 x h1], out [h1 x h1],
                                  * fc1 [h2 x h1], fc2 [h1 x h2] (y = x W^T),
                                  * or NULL (all synthetic)                     */
    const hp_tensor_src* norm;   /* [n_layers*4] LN1 gamma, beta, LN2 gamma,
                                  * beta [h1], or NULL                          */
    hp_tensor_src embed;         /* [vocab x h1] (tied LM head)                 */
    hp_tensor_src pos;           /* [pos_s x h1] learned positions              */
    hp_tensor_src final_norm[2]; /* [h1] gamma, beta                            */
    int64_t bin_bytes;
} hp_weight_set;
hp_status hp_nccl_unique_id(void* out128);
/* weights: NULL = every tensor synthetic (read during the call only).    */
hp_status hp_pipeline_create(const char* plan_json, const char* model_json, int rank,
                             int world, const void* nccl_ids,
                             const hp_pipeline_options* opt, const hp_weight_set* weights,
                             hp_pipeline** out);
/* One serving round: B requests, prompt s, n generated tokens (the plan's
 * workload), greedy decoding. host_tokens (rank 0): [B x s] int32 prompt
 * token ids, or NULL for the device-resident synthetic prompt. host_out
 * (last rank): [B x n] int32 generated token ids, or NULL. timing4 =
 * {makespan_s, prefill_s, decode_s, io_s} of this rank (CUDA events).    */
hp_status hp_pipeline_run(hp_pipeline* p, const int32_t* host_tokens, int32_t* host_out,
                          double* timing4);
/* Last rank: final hidden state (pre final-LN) of every request's last
 * position of the last round, [B x h1] bf16 host buffer.                 */
hp_status hp_pipeline_final_hidden(hp_pipeline* p, void* host);
/* Weight load of hp_pipeline_create: {seconds, source bf16 bytes read,
 * resident bytes, H2D bins}.                                             */
hp_status hp_pipeline_load_stats(hp_pipeline* p, double* out4);
/* Measured mean per-unit costs {pre_s, dec_s, 0, 0} of the last round, for
 * pipesim::simulate (comm costs are the caller's).                      */
hp_status hp_pipeline_stage_costs(hp_pipeline* p, double* out4);
/* Instrumented totals {launches, seconds, algorithmic_bytes, flops}
 * accumulated over rounds; kind 0 = prefill linear ops (K4), 1 = decode
 * linear ops (K3), 2 = prefill attention, 3 = decode attention.          */
hp_status hp_pipeline_kernel_stats(hp_pipeline* p, int kind, double* out4);
/* Per-layer seconds (LN + 4 linear ops) of this stage's layers in the
 * instrumented unit of the last instrument=1 round: one prefill micro-batch
 * (HP_PREFILL) or one decode group-token (HP_DECODE); *n = layer count.   */
hp_status hp_pipeline_layer_costs(hp_pipeline* p, int phase, double* out, int64_t cap,
                                  int64_t* n);
/* {packed weight bytes, kernel launches per round, units, layers}        */
hp_status hp_pipeline_info(hp_pipeline* p, int64_t* out4);
void hp_pipeline_destroy(hp_pipeline* p);

/* ---- micro-batch manager (hetplan::runtime::
 * microbatch_manager): thread-safe status table of one round. prefill_done
 * returns the group it made ready (its first decode token enqueued) or -1;
 * decode_done enqueues the group's next token (*finished = 1 after token
 * n-1); next pops the FIFO of ready decode items (returns 1, or 0 if empty). */
typedef struct hp_mbm hp_mbm;
hp_status hp_mbm_create(int B, int eta, int xi, int n, hp_mbm** out);
hp_status hp_mbm_prefill_done(hp_mbm* m, int k, int* ready_group);
hp_status hp_mbm_decode_done(hp_mbm* m, int group, int token, int* finished);
int hp_mbm_next(hp_mbm* m, int* group, int* token);
void hp_mbm_destroy(hp_mbm* m);

/* ---- host planning helpers (drop-in hetplan:: library, plain types) -----
 * model9 = {num_layers, h1, h2, num_heads, vocab_s, pos_s, d_t, d_p,
 * norm(0 standard, 1 rms)}. Text outputs are NUL-terminated into out/cap.  */
hp_status hp_host_scaling_factor(double w_min, double w_max, int bit, int scheme,
                                 double* out);
hp_status hp_host_g_of_x(double mean, double var, int rounding, double* out);
hp_status hp_host_indicator_csv(const char* stats_csv, const int* bits, int nbits,
                                int scheme, int rounding, char* out, int64_t cap);
/* omega [n_layers × nbits] from per-op stats5 (K2 output layout),
 * ops in qkv,out,fc1,fc2 order (indicator.cpp:99-127 op order).         */
hp_status hp_host_omega_from_stats(const double* stats5_per_op, int n_layers,
                                   int ops_per_layer, const int* bits, int nbits,
                                   int scheme, int rounding, double* omega_out);
/* Monte-Carlo output variance of one operator row (indicator.cpp:231-284,
 * SPEC Theorem 1 check): out4 = {total_var, extra_var, se_total, n}.      */
hp_status hp_host_mc_output_variance(const double* w, int64_t d, double x_mean, double x_var,
                                    int bit, int scheme, int rounding, int64_t n_samples,
                                    uint64_t seed, double* out4);
hp_status hp_host_memcost(const int64_t* model9, int bit, int64_t v, int64_t s,
                          int64_t n, int64_t* out3);
hp_status hp_host_preset(const char* name, int64_t* model9);
hp_status hp_host_make_schedule(int B, int eta, int xi, int* sizes, int* groups,
                                int* n_batches, int* n_groups, int cap);
hp_status hp_host_simulate(const double* costs4, int n_stages, int B, int eta,
                           int xi, int n, double* out4, double* busy,
                           double* timeline, int64_t timeline_cap);
hp_status hp_host_plan_check(const char* plan_json, char* out, int64_t cap);
/* Unit execution order of one stage: (kind 0 prefill / 1 decode, index,
 * token) triples into out3[3*cap]; *n = count.                          */
hp_status hp_host_unit_order(const char* plan_json, const char* model_json, int stage,
                             int* out3, int cap, int* n);
/* Latency model (hetplan::latcost, latcost.cpp:140-225; Eigen-free QR):
 * fit a profile CSV "device,bit,phase,v,s,t,latency_s" into the model JSON
 * (serialize_model, format_version 1) -> out[cap], *needed = bytes incl.
 * the NUL (HP_EINVAL when cap is too small); predict phase 0 prefill(v, s)
 * / 1 decode(v, s, t) from a model JSON.                                   */
hp_status hp_host_latency_fit(const char* profile_csv, char* out, int64_t cap, int64_t* needed);
hp_status hp_host_latency_predict(const char* model_json, const char* device, int bit, int phase,
                                  double v, double s, double t, double* out);

#ifdef __cplusplus
}
#endif
#endif /* HP_CAPI_H */
