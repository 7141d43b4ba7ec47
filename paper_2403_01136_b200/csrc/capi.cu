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
                              double* step64, double* zero64, cudaStream_t st);
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
struct dstage_op {
    const uint8_t* packed;
    const float* scale;
    const float* zero;
    void* y;
    const void* res;
    const CUtensorMap* tmap;
    int64_t ldy, ldr;
    int total;
    int kind;
    int bits, n_out, k_in, G, NT, maxseg, epi, sps;
    unsigned wait;
    const void* ln_x;
    const void* gamma;
    const void* beta;
    void* ln_y;
    int64_t ln_ldx, ln_ldy;
    int h;
    int P;
    const unsigned* dep_flags;
    unsigned* out_flags;
    int dep_off;
    int pbuf;
};
static_assert(sizeof(dstage_op) == 192, "dstage_op layout is shared by k3_stage.cu and capi.cu");
int dstage_grid();
cudaError_t launch_layernorm(const void* x, int64_t ldx, int64_t rows, int h, const void* gamma,
                             const void* beta, void* y, int64_t ldy, cudaStream_t st);
cudaError_t launch_dstage(const dstage_op* ops, int nops, int m, int bits, bool sym,
                          unsigned long long* sync, unsigned long long units, unsigned* const counters[2],
                          float* const partial[2], int grid, cudaStream_t st);
int slices_per_stage(int bits, int bn);
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

int hp_abi_version(void) { return 1; }

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

hp_status hp_quant_pack(const void* w, int64_t n_out, int64_t k_in, int64_t ldw, int bits,
                        int scheme, int rounding, void* packed, float* scale, float* zero,
                        double* step64, double* zero64, hp_stream stream) {
    if (!w || !packed) return fail(HP_EINVAL, "quant_pack: NULL w or packed");
    if (n_out <= 0 || k_in <= 0) return fail(HP_EINVAL, "quant_pack: empty shape");
    if (ldw < k_in) return fail(HP_EINVAL, "quant_pack: ldw < k_in");
    if (!bits_ok(bits)) return fail(HP_EINVAL, "quant_pack: bits must be 3, 4, 8 or 16");
    if (scheme != HP_ASYMMETRIC && scheme != HP_SYMMETRIC)
        return fail(HP_EINVAL, "quant_pack: unknown scheme");
    if (rounding != HP_NEAREST)
        return fail(HP_EINVAL,
                    "quant_pack: only round-to-nearest is supported on the GPU (the "
                    "reference's stochastic rounding draws a sequential mt19937_64 stream)");
    if (bits != 16 && !scale) return fail(HP_EINVAL, "quant_pack: scale is NULL");
    if ((step64 == nullptr) != (zero64 == nullptr))
        return fail(HP_EINVAL, "quant_pack: step64 and zero64 go together");
    if (hp_status s = need_device()) return s;
    return cuda_status(hp::launch_quant_pack(w, n_out, k_in, ldw, bits, scheme, packed, scale,
                                             zero, step64, zero64,
                                             static_cast<cudaStream_t>(stream)),
                       "quant_pack");
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
    if (!w || !stats5) return fail(HP_EINVAL, "indicator_stats: NULL w or stats5");
    if (n_out <= 0 || k_in <= 0) return fail(HP_EINVAL, "indicator_stats: empty weight");
    if (ldw < k_in) return fail(HP_EINVAL, "indicator_stats: ldw < k_in");
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
    const double wb = static_cast<double>(n_out) * k_in, xb = x ? 4.0 * tokens * k_in : 0.0;
    const int nb = 3 * sms;
    const int nbx = x ? std::max(1, std::min(nb - 1, static_cast<int>(nb * xb / (wb + xb)))) : 0;
    const int nbw = std::max(1, nb - nbx);
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

struct hp_decode_plan {
    struct run {  // consecutive layers of one bit width = one kernel launch
        int op0, nops, bits;
        unsigned long long units;
        unsigned long long* sync;
    };
    std::vector<void*> allocs;
    std::vector<run> runs;
    hp::dstage_op* d_ops = nullptr;
    int nops = 0;
    int m = 0;
    bool sym = true;
    unsigned* counters[2] = {nullptr, nullptr};
    float* partial[2] = {nullptr, nullptr};
    int grid = 0;
    double weight_bytes = 0, alg_bytes = 0;
    void* scratch[3] = {nullptr, nullptr, nullptr};
};

/* debug (not in the ABI header): scratch buffers a, qkv, f of a plan */
void hp_decode_plan_debug_scratch(hp_decode_plan* p, void** out3) {
    for (int i = 0; i < 3; ++i) out3[i] = p->scratch[i];
}

hp_status hp_decode_plan_create(const hp_decoder_layer* layers, int n_layers, void* x,
                                int64_t m, hp_decode_plan** out) {
    if (!out) return fail(HP_EINVAL, "decode_plan: NULL out");
    *out = nullptr;
    if (!layers || n_layers <= 0) return fail(HP_EINVAL, "decode_plan: no layers");
    if (!x || (reinterpret_cast<uintptr_t>(x) & 15)) return fail(HP_EINVAL, "decode_plan: x must be 16-byte aligned");
    if (m <= 0 || m > 32) return fail(HP_EINVAL, "decode_plan: m must be in [1, 32]");
    const int64_t h1 = layers[0].ops[1].n_out, h2 = layers[0].ops[2].n_out;
    const int scheme = layers[0].ops[0].scheme;
    if (h1 <= 0 || h1 % 128 || h2 % 128 || h1 > 16384)
        return fail(HP_EINVAL, "decode_plan: h1, h2 must be multiples of 128 (h1 <= 16384)");
    for (int l = 0; l < n_layers; ++l) {
        const hp_decoder_layer& L = layers[l];
        const int64_t shp[4][2] = {{3 * h1, h1}, {h1, h1}, {h2, h1}, {h1, h2}};
        for (int o = 0; o < 4; ++o) {
            if (hp_status s = check_qweight(&L.ops[o])) return s;
            if (L.ops[o].n_out != shp[o][0] || L.ops[o].k_in != shp[o][1])
                return fail(HP_EINVAL, "decode_plan: layer " + std::to_string(l) + " op " +
                                           std::to_string(o) + " has the wrong shape");
            if (L.ops[o].scheme != scheme) return fail(HP_EINVAL, "decode_plan: mixed schemes");
        }
        for (int j = 0; j < 4; ++j)
            if (!L.ln[j] || (reinterpret_cast<uintptr_t>(L.ln[j]) & 15))
                return fail(HP_EINVAL, "decode_plan: LN parameters must be 16-byte aligned");
    }
    if (hp_status s = need_device()) return s;
    auto* p = new hp_decode_plan();
    auto cleanup = [&](hp_status s) {
        hp_decode_plan_destroy(p);
        return s;
    };
    auto dalloc = [&](size_t bytes) -> void* {
        void* q = nullptr;
        if (cudaMalloc(&q, std::max<size_t>(bytes, 256)) != cudaSuccess) return nullptr;
        p->allocs.push_back(q);
        return q;
    };
    p->m = static_cast<int>(m);
    p->sym = scheme == HP_SYMMETRIC;
    p->grid = hp::dstage_grid();
    void* scr_a = dalloc(m * h1 * 2);
    void* scr_qkv = dalloc(m * 3 * h1 * 2);
    void* scr_f = dalloc(m * h2 * 2);
    if (!scr_a || !scr_qkv || !scr_f) return cleanup(fail(HP_ECUDA, "decode_plan: cudaMalloc"));
    p->scratch[0] = scr_a;
    p->scratch[1] = scr_qkv;
    p->scratch[2] = scr_f;
    // host op table + tensor maps
    std::vector<hp::dstage_op> ops;
    std::vector<CUtensorMap> maps;
    std::vector<int> map_of;  // op index -> map index
    std::vector<std::pair<int, int>> flag_of;  // op index -> (flags offset, count) or (-1, 0)
    size_t part_bytes = 0;
    int max_nt = 1, nflags = 0, ngemm = 0;
    unsigned done = 0;  // units of the current run so far
    auto gemm = [&](const hp_qweight& w, const void* xin, int64_t ldx, void* y, int64_t ldy,
                    const void* res, int epi, bool flags_out, int dep_op, int dep_off) -> hp_status {
        hp::dstage_op op{};
        op.kind = 0;
        op.bits = w.bits;
        op.packed = static_cast<const uint8_t*>(w.packed);
        op.scale = w.scale;
        op.zero = w.zero;
        op.n_out = static_cast<int>(w.n_out);
        op.k_in = static_cast<int>(w.k_in);
        op.G = static_cast<int>(hp::ceil_div64(w.k_in, 128));
        op.NT = static_cast<int>(hp::ceil_div64(w.n_out, 128));
        op.total = op.NT * op.G;
        const int64_t grid = std::min<int64_t>(p->grid, op.total);
        op.P = static_cast<int>(grid);
        const int64_t per = op.total / grid;
        op.maxseg = static_cast<int>(std::min<int64_t>((op.G + per - 1) / per + 1, grid));
        op.sps = w.bits <= 4 ? 8 : (w.bits == 8 ? 4 : 2);
        op.y = y;
        op.ldy = ldy;
        op.res = res;
        op.ldr = res ? ldy : 0;
        op.epi = epi;
        op.wait = done;
        op.pbuf = (ngemm++) & 1;
        op.dep_off = dep_off;
        done += static_cast<unsigned>(op.NT);
        CUtensorMap map;
        if (hp_status s = make_act_map(&map, xin, w.k_in, m, ldx, 32, op.sps / 2)) return s;
        map_of.push_back(static_cast<int>(maps.size()));
        maps.push_back(map);
        // flags resolved to device pointers after the upload
        flag_of.push_back(flags_out ? std::make_pair(nflags, op.NT) : std::make_pair(-1, dep_op));
        if (flags_out) nflags += op.NT;
        ops.push_back(op);
        part_bytes = std::max(part_bytes, static_cast<size_t>(op.NT) * op.maxseg * 128 * 32 * 4);
        max_nt = std::max(max_nt, op.NT);
        p->weight_bytes += static_cast<double>(hp_packed_bytes(w.n_out, w.k_in, w.bits)) +
                           (w.bits == 16 ? 0.0 : 4.0 * hp_scale_count(w.n_out, w.k_in) *
                                                     (w.scheme == HP_SYMMETRIC ? 1 : 2));
        p->alg_bytes += 2.0 * m * (w.n_out + w.k_in);
        return HP_OK;
    };
    auto ln = [&](const void* gamma, const void* beta) {
        hp::dstage_op op{};
        op.kind = 1;
        op.ln_x = x;
        op.ln_ldx = h1;
        op.ln_y = scr_a;
        op.ln_ldy = h1;
        op.gamma = gamma;
        op.beta = beta;
        op.h = static_cast<int>(h1);
        op.wait = done;
        done += static_cast<unsigned>(m);
        map_of.push_back(-1);
        flag_of.push_back({-1, -1});
        ops.push_back(op);
    };
    std::vector<int> dep_of;  // op -> producing op index for dataflow edges (or -1)
    for (int l = 0; l < n_layers; ++l) {
        const hp_decoder_layer& L = layers[l];
        if (l == 0 || L.ops[0].bits != layers[l - 1].ops[0].bits) {  // new run: a kernel boundary
            if (!p->runs.empty()) {
                p->runs.back().nops = static_cast<int>(ops.size()) - p->runs.back().op0;
                p->runs.back().units = done;
            }
            p->runs.push_back({static_cast<int>(ops.size()), 0, L.ops[0].bits, 0, nullptr});
            done = 0;
        }
        for (int o = 1; o < 4; ++o)
            if (L.ops[o].bits != L.ops[0].bits)
                return cleanup(fail(HP_EINVAL, "decode_plan: the four ops of a layer must share a bit width"));
        const int i0 = static_cast<int>(ops.size());
        ln(L.ln[0], L.ln[1]);
        if (hp_status s = gemm(L.ops[0], scr_a, h1, scr_qkv, 3 * h1, nullptr, 0, true, -1, 0)) return cleanup(s);
        // out-proj reads the V slice: qkv output tiles [2 h1/128, 3 h1/128)
        if (hp_status s = gemm(L.ops[1], static_cast<char*>(scr_qkv) + 2 * h1 * 2, 3 * h1, x, h1, x, 0, false,
                               i0 + 1, static_cast<int>(2 * h1 / 128)))
            return cleanup(s);
        ln(L.ln[2], L.ln[3]);
        if (hp_status s = gemm(L.ops[2], scr_a, h1, scr_f, h2, nullptr, HP_EPI_RELU, true, -1, 0)) return cleanup(s);
        if (hp_status s = gemm(L.ops[3], scr_f, h2, x, h1, x, 0, false, i0 + 4, 0)) return cleanup(s);
    }
    p->runs.back().nops = static_cast<int>(ops.size()) - p->runs.back().op0;
    p->runs.back().units = done;
    p->alg_bytes += p->weight_bytes;
    p->nops = static_cast<int>(ops.size());
    // device image: [maps (64-B aligned)] [ops] [sync per run] [flags] [tickets x2] [partials x2]
    auto up = [](size_t v) { return (v + 255) / 256 * 256; };
    const size_t maps_bytes = maps.size() * sizeof(CUtensorMap);
    const size_t ops_off = up(maps_bytes);
    const size_t ops_bytes = ops.size() * sizeof(hp::dstage_op);
    const size_t sync_off = up(ops_off + ops_bytes);
    const size_t sync_bytes = p->runs.size() * 256;
    const size_t flags_off = up(sync_off + sync_bytes);
    const size_t flags_bytes = static_cast<size_t>(nflags) * 4;
    const size_t tick_off = up(flags_off + flags_bytes);
    const size_t tick_bytes = up(static_cast<size_t>(max_nt) * 4);
    const size_t part_off = up(tick_off + 2 * tick_bytes);
    auto* base = static_cast<char*>(dalloc(part_off + 2 * part_bytes));
    if (!base) return cleanup(fail(HP_ECUDA, "decode_plan: cudaMalloc"));
    auto* dmaps = reinterpret_cast<CUtensorMap*>(base);
    auto* dflags = reinterpret_cast<unsigned*>(base + flags_off);
    for (size_t i = 0; i < ops.size(); ++i) {
        if (map_of[i] >= 0) ops[i].tmap = dmaps + map_of[i];
        if (ops[i].kind == 0 && flag_of[i].first >= 0) ops[i].out_flags = dflags + flag_of[i].first;
    }
    for (size_t i = 0; i < ops.size(); ++i) {  // dataflow edges: the producer's flags
        if (ops[i].kind == 0 && flag_of[i].first < 0 && flag_of[i].second >= 0)
            ops[i].dep_flags = ops[flag_of[i].second].out_flags;
    }
    for (size_t r = 0; r < p->runs.size(); ++r)
        p->runs[r].sync = reinterpret_cast<unsigned long long*>(base + sync_off + r * 256);
    p->d_ops = reinterpret_cast<hp::dstage_op*>(base + ops_off);
    for (int b = 0; b < 2; ++b) {
        p->counters[b] = reinterpret_cast<unsigned*>(base + tick_off + b * tick_bytes);
        p->partial[b] = reinterpret_cast<float*>(base + part_off + b * part_bytes);
    }
    if (cudaMemcpy(dmaps, maps.data(), maps_bytes, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(p->d_ops, ops.data(), ops_bytes, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemset(base + sync_off, 0, part_off - sync_off) != cudaSuccess)
        return cleanup(fail(HP_ECUDA, "decode_plan: upload"));
    *out = p;
    return HP_OK;
}

hp_status hp_decode_plan_run(hp_decode_plan* p, hp_stream stream) {
    if (!p) return fail(HP_EINVAL, "decode_plan_run: NULL plan");
    int limit = p->nops;
    if (const char* e = getenv("HP_DSTAGE_NOPS")) limit = std::min(limit, atoi(e));  // debug
    for (const auto& r : p->runs) {
        const int n = std::min(r.nops, limit - r.op0);
        if (n <= 0) break;
        // a truncated run (debug) must still see its full per-launch unit count
        // only when complete; recompute for the prefix
        unsigned long long units = r.units;
        if (n < r.nops) {
            std::vector<hp::dstage_op> tmp(1);
            cudaMemcpy(tmp.data(), p->d_ops + r.op0 + n, sizeof(hp::dstage_op), cudaMemcpyDeviceToHost);
            units = tmp[0].wait;
        }
        if (hp_status s = cuda_status(
                hp::launch_dstage(p->d_ops + r.op0, n, p->m, r.bits, p->sym, r.sync, units, p->counters,
                                  p->partial, p->grid, static_cast<cudaStream_t>(stream)),
                "decode_plan_run"))
            return s;
    }
    return HP_OK;
}

hp_status hp_decode_plan_info(hp_decode_plan* p, double* out4) {
    if (!p || !out4) return fail(HP_EINVAL, "decode_plan_info: NULL argument");
    out4[0] = p->weight_bytes;
    out4[1] = p->alg_bytes;
    out4[2] = p->nops;
    out4[3] = p->grid;
    return HP_OK;
}

void hp_decode_plan_destroy(hp_decode_plan* p) {
    if (!p) return;
    for (void* q : p->allocs) cudaFree(q);
    delete p;
}

}  // extern "C"
