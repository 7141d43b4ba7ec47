// C-ABI entry points (include/hp_capi.h): argument validation, error
// mapping (exceptions never cross the ABI), TMA descriptor encoding and
// kernel dispatch. No CPU fallback: without a usable sm_100 device every
// compute entry point fails with HP_ECUDA.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>
#include <algorithm>

#include "hp_capi.h"
#include "layout.cuh"

namespace hp {
extern int g_sm_budget;
extern int g_pdl;
extern unsigned long long* g_trace;
cudaError_t launch_quant_pack(const void* w, int64_t n_out, int64_t k_in, int64_t ldw,
                              int bits, int sym, void* packed, float* scale, float* zero,
                              double* step64, double* zero64, double* stats5, cudaStream_t st);
cudaError_t launch_unpack(const void* packed, const float* scale, const float* zero,
                          int64_t n_out, int64_t k_in, int bits, void* codes,
                          float* scale_rm, float* zero_rm, cudaStream_t st);
cudaError_t launch_dequant(const void* packed, const float* scale, const float* zero,
                           int64_t n_out, int64_t k_in, int bits, int sym, void* out,
                           cudaStream_t st);
size_t stats_scratch_bytes(int nbw, int nbx);
cudaError_t launch_stats(const void* w, int64_t n_out, int64_t k_in, int64_t ldw,
                         const void* x, int64_t tokens, int64_t ldx, double* out,
                         void* scratch, int nbw, int nbx, cudaStream_t st);
struct qgemm_plan {
    int bn, mt, splits, gps, units, grid;
    size_t workspace;
    int stream_k, maxseg;
    int64_t total;
    int dp;
};
qgemm_plan plan_qgemm(int64_t n_out, int64_t k_in, int64_t m, int phase);
int slices_per_stage(int bits, int bn);
cudaError_t launch_layernorm(const void* x, int64_t ldx, int64_t rows, int h, const void* gamma,
                             const void* beta, void* y, int64_t ldy, cudaStream_t st);
cudaError_t launch_embed(const int32_t* tok, int rows, int pos0, int pos_per_req, int s_tokens,
                         const void* E, const void* P, int pos_s, int h, int64_t vocab, void* x,
                         cudaStream_t st);
cudaError_t launch_attn_prefill(const void* qkv, int reqs, int s, int h, int D, void* out, void* kc,
                                void* vc, int req0, int S_max, cudaStream_t st);
cudaError_t launch_attn_decode(const void* qkv, int rows, int h, int D, int p, void* out, void* kc,
                               void* vc, int req0, int S_max, cudaStream_t st, void* ws, int split);
size_t attn_decode_workspace(int rows, int h, int D, int split);
cudaError_t launch_argmax(const void* logits, int64_t ld, int rows, int64_t vocab, int32_t* tok,
                          int32_t* tok2, int64_t tok2_stride, cudaStream_t st);
cudaError_t launch_qgemm(const CUtensorMap& map, const qgemm_plan& p, int bits, bool sym,
                         const void* packed, const float* scale, const float* zero,
                         int64_t n_out, int64_t k_in, int64_t m, void* y, int64_t ldy,
                         const void* res, int64_t ldr, int epi, void* workspace,
                         cudaStream_t st);
}  // namespace hp

namespace {
thread_local std::string g_error;
}  // namespace

namespace hp_detail {
void set_error(const std::string& msg) { g_error = msg; }
}  // namespace hp_detail

namespace {

hp_status fail(hp_status s, const std::string& msg) {
    g_error = msg;
    return s;
}

hp_status cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return HP_OK;
    return fail(HP_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

bool bits_ok(int b) { return b == 3 || b == 4 || b == 8 || b == 16; }

int device_ok_cached() {
    static int ok = -1;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (ok < 0) {
        int dev = 0, major = 0;
        ok = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) ==
                cudaSuccess &&
            major == 10)
            ok = 1;
        cudaGetLastError();
    }
    return ok;
}

hp_status need_device() {
    if (!device_ok_cached())
        return fail(HP_ECUDA, "no usable sm_100 (B200) device; the CPU path is not a fallback");
    return HP_OK;
}

using encode_fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                               const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                               const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

encode_fn get_encode() {
    static encode_fn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<encode_fn>(p);
        cudaGetLastError();
    });
    return fn;
}

// Activations [rows × k] bf16, row stride ld elements, viewed as 3-D
// {64 k, rows, k/64 slices}: one TMA box {64, box_rows, slices} lands
// `slices` consecutive [box_rows × 64] sub-tiles, each in the UMMA K-major
// 128-byte-swizzle layout. OOB (ragged k / rows) -> zero.
hp_status make_act_map(CUtensorMap* map, const void* x, int64_t k, int64_t rows,
                       int64_t ld, int box_rows, int slices) {
    encode_fn enc = get_encode();
    if (!enc) return fail(HP_ECUDA, "cuTensorMapEncodeTiled unavailable");
    // innermost dim covers exactly 64 elements per slice; k padded to 64
    const int64_t nslices = (k + 63) / 64;
    cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(nslices)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 2, 128};
    cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(slices)};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(x), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(HP_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    return HP_OK;
}

hp_status check_qweight(const hp_qweight* w) {
    if (!w) return fail(HP_EINVAL, "qweight is NULL");
    if (w->n_out <= 0 || w->k_in <= 0) return fail(HP_EINVAL, "qweight: empty shape");
    if (!bits_ok(w->bits)) return fail(HP_EINVAL, "qweight: bits must be 3, 4, 8 or 16");
    if (w->scheme != HP_ASYMMETRIC && w->scheme != HP_SYMMETRIC)
        return fail(HP_EINVAL, "qweight: unknown scheme");
    if (!w->packed) return fail(HP_EINVAL, "qweight: packed is NULL");
    if (w->bits != 16 && !w->scale) return fail(HP_EINVAL, "qweight: scale is NULL");
    if (w->bits != 16 && w->scheme == HP_ASYMMETRIC && !w->zero)
        return fail(HP_EINVAL, "qweight: asymmetric weights need zero");
    if (w->n_out > (1LL << 30) || w->k_in > (1LL << 30))
        return fail(HP_EINVAL, "qweight: dimension too large");
    return HP_OK;
}

}  // namespace

extern "C" {

const char* hp_last_error(void) { return g_error.c_str(); }

int hp_abi_version(void) { return 2; }

int hp_device_ok(void) { return device_ok_cached(); }

void hp_set_sm_budget(int sms) { hp::g_sm_budget = sms > 0 ? sms : 0; }

void hp_set_pdl(int enable) { hp::g_pdl = enable ? 1 : 0; }

/* debug: copy the HP_QGEMM_TRACE clock trace (4 roles x 64 iters x 4 events) */
int hp_debug_trace(unsigned long long* host, int n) {
    if (!hp::g_trace) return 0;
    cudaDeviceSynchronize();
    cudaMemcpy(host, hp::g_trace, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost);
    return n;
}

int64_t hp_packed_bytes(int64_t n_out, int64_t k_in, int bits) {
    if (n_out <= 0 || k_in <= 0 || !bits_ok(bits)) return -1;
    return hp::ceil_div64(n_out, 128) * hp::ceil_div64(k_in, 128) * hp::tile_bytes(bits);
}

int64_t hp_scale_count(int64_t n_out, int64_t k_in) {
    if (n_out <= 0 || k_in <= 0) return -1;
    return hp::ceil_div64(n_out, 128) * hp::ceil_div64(k_in, 128) * 128;
}

static hp_status quant_pack_impl(const char* who, const void* w, int64_t n_out, int64_t k_in,
                                 int64_t ldw, int bits, int scheme, int rounding, void* packed,
                                 float* scale, float* zero, double* step64, double* zero64,
                                 double* stats5, hp_stream stream) {
    if (!w || !packed) return fail(HP_EINVAL, std::string(who) + ": NULL w or packed");
    if (n_out <= 0 || k_in <= 0) return fail(HP_EINVAL, std::string(who) + ": empty shape");
    if (ldw < k_in) return fail(HP_EINVAL, std::string(who) + ": ldw < k_in");
    if (!bits_ok(bits)) return fail(HP_EINVAL, std::string(who) + ": bits must be 3, 4, 8 or 16");
    if (scheme != HP_ASYMMETRIC && scheme != HP_SYMMETRIC)
        return fail(HP_EINVAL, std::string(who) + ": unknown scheme");
    if (rounding != HP_NEAREST)
        return fail(HP_EINVAL, std::string(who) +
                                   ": only round-to-nearest is supported on the GPU (the "
                                   "reference's stochastic rounding draws a sequential mt19937_64 stream)");
    if (bits != 16 && !scale) return fail(HP_EINVAL, std::string(who) + ": scale is NULL");
    if ((step64 == nullptr) != (zero64 == nullptr))
        return fail(HP_EINVAL, std::string(who) + ": step64 and zero64 go together");
    if (n_out >= (int64_t(1) << 31) || k_in >= (int64_t(1) << 31))
        return fail(HP_EINVAL, std::string(who) + ": n_out and k_in must be < 2^31");
    if (hp_status s = need_device()) return s;
    return cuda_status(hp::launch_quant_pack(w, n_out, k_in, ldw, bits, scheme, packed, scale,
                                             zero, step64, zero64, stats5,
                                             static_cast<cudaStream_t>(stream)),
                       who);
}

hp_status hp_quant_pack(const void* w, int64_t n_out, int64_t k_in, int64_t ldw, int bits,
                        int scheme, int rounding, void* packed, float* scale, float* zero,
                        double* step64, double* zero64, hp_stream stream) {
    return quant_pack_impl("quant_pack", w, n_out, k_in, ldw, bits, scheme, rounding, packed, scale,
                           zero, step64, zero64, nullptr, stream);
}

hp_status hp_quant_pack_stats(const void* w, int64_t n_out, int64_t k_in, int64_t ldw, int bits,
                              int scheme, int rounding, void* packed, float* scale, float* zero,
                              double* step64, double* zero64, double* stats5, hp_stream stream) {
    if (!stats5) return fail(HP_EINVAL, "quant_pack_stats: NULL stats5");
    return quant_pack_impl("quant_pack_stats", w, n_out, k_in, ldw, bits, scheme, rounding, packed,
                           scale, zero, step64, zero64, stats5, stream);
}

hp_status hp_quant_unpack(const hp_qweight* w, void* codes, float* scale_rm, float* zero_rm,
                          hp_stream stream) {
    if (hp_status s = check_qweight(w)) return s;
    if (hp_status s = need_device()) return s;
    return cuda_status(hp::launch_unpack(w->packed, w->scale, w->zero, w->n_out, w->k_in,
                                         w->bits, codes, scale_rm, zero_rm,
                                         static_cast<cudaStream_t>(stream)),
                       "quant_unpack");
}

hp_status hp_dequant(const hp_qweight* w, void* w_bf16, hp_stream stream) {
    if (hp_status s = check_qweight(w)) return s;
    if (!w_bf16) return fail(HP_EINVAL, "dequant: NULL output");
    if (hp_status s = need_device()) return s;
    return cuda_status(hp::launch_dequant(w->packed, w->scale, w->zero, w->n_out, w->k_in,
                                          w->bits, w->scheme == HP_SYMMETRIC, w_bf16,
                                          static_cast<cudaStream_t>(stream)),
                       "dequant");
}

// One memory pool per device for small stream-ordered scratch, with an
// unbounded release threshold so freed blocks are reused, never unmapped.
static cudaMemPool_t scratch_pool() {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if (cudaMemPoolCreate(&pools[dev], &props) != cudaSuccess) {
            cudaGetLastError();
            cudaDeviceGetDefaultMemPool(&pools[dev], dev);
        }
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
    }
    return pools[dev];
}

hp_status hp_indicator_stats(const void* w, int64_t n_out, int64_t k_in, int64_t ldw,
                             const void* x, int64_t tokens, int64_t ldx, double* stats5,
                             hp_stream stream) {
    if (!stats5) return fail(HP_EINVAL, "indicator_stats: NULL stats5");
    if (!w && !x) return fail(HP_EINVAL, "indicator_stats: NULL w and x");
    if (k_in <= 0) return fail(HP_EINVAL, "indicator_stats: empty k_in");
    if (w && (n_out <= 0 || ldw < k_in)) return fail(HP_EINVAL, "indicator_stats: bad weight shape");
    if (x && (tokens <= 0 || ldx < k_in))
        return fail(HP_EINVAL, "indicator_stats: bad calibration shape");
    if (hp_status s = need_device()) return s;
    auto st = static_cast<cudaStream_t>(stream);
    // 3 resident blocks of 256 threads per SM (one wave), split between W and X by cost
    int sms = 148;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    // (an X element costs ~4x a W element: fp64 moments vs fp32 min/max, so
    // X blocks get proportionally fewer bytes and finish with the W blocks)
    // w == NULL: the weight part was produced by hp_quant_pack_stats (K1's
    // fused pass); only stats5[3..4] are written
    const double wb = w ? static_cast<double>(n_out) * k_in : 0.0, xb = x ? 4.0 * tokens * k_in : 0.0;
    const int nb = 3 * sms;
    const int nbx = !x ? 0 : (!w ? nb : std::max(1, std::min(nb - 1, static_cast<int>(nb * xb / (wb + xb)))));
    const int nbw = !w ? 0 : std::max(1, nb - nbx);
    const size_t bytes = hp::stats_scratch_bytes(nbw, nbx);
    void* scratch = nullptr;
    // stream-ordered scratch from a private pool that keeps its memory: a
    // default-pool cudaMallocAsync/cudaFreeAsync pair re-maps physical pages
    // at every synchronisation (~2 ms per call, 30x the kernel itself)
    cudaError_t e = cudaMallocFromPoolAsync(&scratch, bytes, scratch_pool(), st);
    if (e != cudaSuccess) return cuda_status(e, "indicator_stats alloc");
    e = cudaMemsetAsync(scratch, 0, 256, st);
    if (e == cudaSuccess)
        e = hp::launch_stats(w, n_out, k_in, ldw, x, tokens, ldx, stats5, scratch, nbw, nbx, st);
    cudaFreeAsync(scratch, st);
    return cuda_status(e, "indicator_stats");
}

size_t hp_qlinear_workspace_bytes(const hp_qweight* w, int64_t m, int phase) {
    if (!w || w->n_out <= 0 || w->k_in <= 0 || m <= 0) return 0;
    return hp::plan_qgemm(w->n_out, w->k_in, m, phase).workspace;
}

hp_status hp_qlinear(const hp_qweight* w, const void* x, int64_t ldx, int64_t m, void* y,
                     int64_t ldy, const void* residual, int64_t ldr, int epilogue, int phase,
                     void* workspace, size_t workspace_bytes, hp_stream stream) {
    if (hp_status s = check_qweight(w)) return s;
    if (m <= 0) return fail(HP_EINVAL, "qlinear: m must be positive");
    if (!x || !y) return fail(HP_EINVAL, "qlinear: NULL x or y");
    if (ldx < w->k_in || ldx % 8 != 0 || (reinterpret_cast<uintptr_t>(x) & 15))
        return fail(HP_EINVAL, "qlinear: x must be 16-byte aligned with ldx >= k_in, ldx % 8 == 0");
    if (ldy < w->n_out) return fail(HP_EINVAL, "qlinear: ldy < n_out");
    if (residual && ldr < w->n_out) return fail(HP_EINVAL, "qlinear: ldr < n_out");
    if (phase != HP_PREFILL && phase != HP_DECODE) return fail(HP_EINVAL, "qlinear: bad phase");
    if (epilogue & ~HP_EPI_RELU) return fail(HP_EINVAL, "qlinear: unknown epilogue flags");
    if (m > (1LL << 30)) return fail(HP_EINVAL, "qlinear: m too large");
    if (hp_status s = need_device()) return s;
    const hp::qgemm_plan p = hp::plan_qgemm(w->n_out, w->k_in, m, phase);
    if (p.workspace > 0 && (workspace == nullptr || workspace_bytes < p.workspace))
        return fail(HP_EINVAL, "qlinear: workspace too small (need " +
                                   std::to_string(p.workspace) + " bytes)");
    CUtensorMap map;
    if (hp_status s = make_act_map(&map, x, w->k_in, m, ldx, p.bn, hp::slices_per_stage(w->bits, p.bn) / 2))
        return s;
    return cuda_status(hp::launch_qgemm(map, p, w->bits, w->scheme == HP_SYMMETRIC, w->packed,
                                        w->scale, w->zero, w->n_out, w->k_in, m, y, ldy,
                                        residual, ldr, epilogue, workspace,
                                        static_cast<cudaStream_t>(stream)),
                       "qlinear");
}

hp_status hp_layernorm(const void* x, int64_t ldx, int64_t rows, int64_t h, const void* gamma,
                       const void* beta, void* y, int64_t ldy, hp_stream stream) {
    if (!x || !gamma || !beta || !y) return fail(HP_EINVAL, "layernorm: NULL pointer");
    if (rows <= 0 || h <= 0 || h > 16384 || ldx < h || ldy < h)
        return fail(HP_EINVAL, "layernorm: bad shape");
    if (hp_status s = need_device()) return s;
    return cuda_status(hp::launch_layernorm(x, ldx, rows, static_cast<int>(h), gamma, beta, y, ldy,
                                            static_cast<cudaStream_t>(stream)),
                       "layernorm");
}

hp_status hp_embed(const int32_t* tok, int rows, int pos0, int pos_per_req, int s_tokens,
                   const void* E, const void* P, int64_t pos_s, int64_t h, int64_t vocab, void* x,
                   hp_stream stream) {
    if (!tok || !E || !x) return fail(HP_EINVAL, "embed: NULL pointer");
    if (rows <= 0 || h <= 0 || h % 8 || vocab <= 0 || (pos_per_req && s_tokens <= 0))
        return fail(HP_EINVAL, "embed: bad shape");
    if (hp_status s = need_device()) return s;
    return cuda_status(hp::launch_embed(tok, rows, pos0, pos_per_req, s_tokens, E, P,
                                        static_cast<int>(pos_s), static_cast<int>(h), vocab, x,
                                        static_cast<cudaStream_t>(stream)),
                       "embed");
}

hp_status hp_attention_prefill(const void* qkv, int reqs, int s, int64_t h, int hd, void* out,
                               void* k_cache, void* v_cache, int req0, int s_max, hp_stream stream) {
    if (!qkv || !out || !k_cache || !v_cache) return fail(HP_EINVAL, "attention_prefill: NULL pointer");
    if ((hd != 64 && hd != 128) || h % hd || reqs <= 0 || s <= 0 || s > s_max || req0 < 0)
        return fail(HP_EINVAL, "attention_prefill: bad shape (head dim 64 or 128)");
    if (hp_status st = need_device()) return st;
    return cuda_status(hp::launch_attn_prefill(qkv, reqs, s, static_cast<int>(h), hd, out, k_cache,
                                               v_cache, req0, s_max, static_cast<cudaStream_t>(stream)),
                       "attention_prefill");
}

size_t hp_attention_decode_workspace_bytes(int rows, int64_t h, int hd, int split) {
    if ((hd != 64 && hd != 128) || h % hd || rows <= 0 || split < 1) return 0;
    return hp::attn_decode_workspace(rows, static_cast<int>(h), hd, split);
}

hp_status hp_attention_decode(const void* qkv, int rows, int64_t h, int hd, int p, void* out,
                              void* k_cache, void* v_cache, int req0, int s_max, int split,
                              void* workspace, size_t ws_bytes, hp_stream stream) {
    if (!qkv || !out || !k_cache || !v_cache) return fail(HP_EINVAL, "attention_decode: NULL pointer");
    if ((hd != 64 && hd != 128) || h % hd || rows <= 0 || p < 0 || p >= s_max || req0 < 0 || split < 1 || split > 8)
        return fail(HP_EINVAL, "attention_decode: bad shape (head dim 64 or 128, split 1..8)");
    if (split > 1 && (!workspace || ws_bytes < hp::attn_decode_workspace(rows, static_cast<int>(h), hd, split)))
        return fail(HP_EINVAL, "attention_decode: split > 1 needs hp_attention_decode_workspace_bytes of zeroed workspace");
    if (hp_status st = need_device()) return st;
    return cuda_status(hp::launch_attn_decode(qkv, rows, static_cast<int>(h), hd, p, out, k_cache,
                                              v_cache, req0, s_max, static_cast<cudaStream_t>(stream),
                                              workspace, split),
                       "attention_decode");
}

hp_status hp_argmax(const void* logits, int64_t ld, int rows, int64_t vocab, int32_t* tok,
                    hp_stream stream) {
    if (!logits || !tok) return fail(HP_EINVAL, "argmax: NULL pointer");
    if (rows <= 0 || vocab <= 0 || ld < vocab || vocab > (int64_t(1) << 31))
        return fail(HP_EINVAL, "argmax: bad shape");
    if (hp_status st = need_device()) return st;
    return cuda_status(hp::launch_argmax(logits, ld, rows, vocab, tok, nullptr, 0,
                                         static_cast<cudaStream_t>(stream)),
                       "argmax");
}

}  // extern "C"
