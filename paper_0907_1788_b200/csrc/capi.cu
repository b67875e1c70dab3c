// capi.cu -- the extern "C" boundary (include/fntrs_gpu.h).
//
// Host-side responsibilities only: argument validation with the reference's
// error classes, plan storage, kernel launches, and canonical ordering of
// escape lists (a CUB radix sort of the few escaped symbol indices). All
// codec arithmetic runs in the CUDA kernels; there is no CPU path.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <map>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fntrs_gpu.h"
#include "field.cuh"
#include "internal.h"

using namespace fntrs_gpu;

struct fntrs_ctx {
    int device = 0;
    Tables tab;
    fast::FastTables ftab;
    bool fast_enabled = true;
    cudaStream_t internal = nullptr;
    uint64_t launches = 0;
    uint64_t fnt_counts[17] = {};  // transforms executed, by log2 size (fntrs_gpu_transform_counts)
    std::string err;
    fast::LogTables ltab;
    std::map<std::pair<uint32_t, uint32_t>, uint32_t*> digit_spectra;  // (N, w) -> Dh [N][D]
    std::map<std::pair<uint32_t, uint32_t>, fntrs_plans*> sys_plans;    // (k, n) -> plan of positions 0..k-1
};

struct fntrs_plans {
    int device = 0;
    cudaStream_t stream = nullptr;  // buffers are stream-ordered allocations on this stream
    uint32_t k = 0, n = 0, N = 0, M = 0, kp = 0, np = 0;
    uint32_t* pos = nullptr;
    uint32_t* ainv = nullptr;
    uint32_t* ahat = nullptr;
    uint32_t ninv = 1;
    uint2* rowmap = nullptr;  // fast-path tables (N == M, kp == k), and the general column path
    uint2* ahat2 = nullptr;
    uint2* sys_w = nullptr;  // systematic conv form: {ahat_j r^-j} Shoup pairs, natural order (fused plans, N <= 4096)
    bool cols = false;        // served by the general column path (codec_cols.cu)
    bool full = false;        // complete reception
    bool split = false;       // 2k > 65536: locator halves' spectra (alo, ahi), product_size 0
    bool gen = false;         // fused M != N decode (codec_gen.cu): rowmap + ahat2 natural pairs
    uint32_t* alo = nullptr;  // [65536][np]
    uint32_t* ahi = nullptr;
};

namespace {

const char* kVersion = "fntrs_b200 0.1 (sm_100a)";

// The fused, generic-fused and four-step kernels form per-stripe symbol
// offsets row * L + col in 32 bits (one IMAD on the multiplier-bound path);
// a stripe whose rows * L reaches 2^32 goes to the tile or column kernels,
// whose offsets are 64-bit.
bool narrow_rows(uint32_t rows, uint32_t L) { return uint64_t(rows) * L < (uint64_t(1) << 32); }

// The transforms a launch executed: `count` transforms of size m (power of two).
void note_fnt(fntrs_ctx* ctx, uint32_t m, uint64_t count) {
    int e = 0;
    while (e < 16 && (1u << e) < m) ++e;
    ctx->fnt_counts[e] += count;
}

// Per-codeword schedule of the decode kernels for a plan (every kernel family
// computes the same transforms; interp.cpp:103-137): complete reception is one
// inverse FNT_N; otherwise FNT1 = FNT_N of N', FNT2 = FNT_M of the truncated
// series, the unscaled inverse FNT_M of the product -- and with 2k > 65536 the
// product by halves: the spectra of S_lo and S_hi and two inverses (size 65536).
void note_decode_schedule(fntrs_ctx* ctx, const fntrs_plans* pl, uint64_t codewords);

uint32_t next_pow2(uint32_t n) {
    uint32_t m = 1;
    while (m < n) m <<= 1;
    return m;
}

int cuda_fail(fntrs_ctx* ctx, cudaError_t e, const char* where) {
    if (ctx) ctx->err = std::string(where) + ": " + cudaGetErrorString(e);
    return FNTRS_E_CUDA;
}

int fail(fntrs_ctx* ctx, int status, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return status;
}

#define CK(call, where)                                   \
    do {                                                  \
        cudaError_t _e = (call);                          \
        if (_e != cudaSuccess) return cuda_fail(ctx, _e, where); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};


// Small escape buffers: one CTA sorts them in shared memory (bitonic network).
// The kernel reads the device-side escape count, so it sorts only the next
// power of two above min(count, cap) -- past the count the buffer already
// holds the ~0 fill -- in one launch instead of the radix sort's several.
constexpr uint32_t kSmallSort = 16384;  // 128 KB of 64-bit keys
__global__ void __launch_bounds__(1024) small_sort_kernel(unsigned long long* keys,
                                                          const unsigned long long* count, uint32_t cap) {
    extern __shared__ unsigned long long s[];
    const unsigned long long c = *count;
    const uint32_t live = c < cap ? uint32_t(c) : cap;
    if (live <= 1) return;
    uint32_t m = 2;
    while (m < live) m <<= 1;
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) s[i] = i < live ? keys[i] : ~0ull;
    __syncthreads();
    for (uint32_t size = 2; size <= m; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < m / 2; i += blockDim.x) {
                const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const unsigned long long a = s[lo], b = s[hi];
                if ((a > b) == up) {
                    s[lo] = b;
                    s[hi] = a;
                }
            }
            __syncthreads();
        }
    for (uint32_t i = threadIdx.x; i < live; i += blockDim.x) keys[i] = s[i];
}

// Larger escape lists: our own merge sort over the live keys [0, min(count,
// cap)) (the device-side count is read by the kernels, so no host sync):
// tiles of kTile keys are sorted in shared memory (bitonic), then runs are
// merged pairwise by merge path -- every CTA owns kMTile consecutive outputs of
// a merged pair, finds where they start in the two runs by a diagonal binary
// search, stages both pieces in shared memory and merges them, each thread
// again splitting its kMergePer outputs by a diagonal search. The passes the
// capacity could need are launched; a pass whose run width already covers the
// live keys exits at once, and a last kernel moves the result back into the
// caller's buffer if it ended in the scratch one. Keys are distinct symbol
// indices, so stability does not matter.
constexpr uint32_t kTile = 4096, kSortThreads = 512, kMTile = 2048, kMergePer = kMTile / kSortThreads;

__device__ __forceinline__ uint32_t live_keys(const unsigned long long* count, uint64_t cap) {
    const unsigned long long c = *count;
    return uint32_t(c < cap ? c : cap);
}

__global__ void __launch_bounds__(kSortThreads) tile_sort_kernel(unsigned long long* keys,
                                                                 const unsigned long long* count, uint64_t cap) {
    __shared__ unsigned long long s[kTile];
    const uint32_t live = live_keys(count, cap), t0 = blockIdx.x * kTile;
    if (t0 >= live || live <= 1) return;
    const uint32_t n = min(kTile, live - t0);
    for (uint32_t i = threadIdx.x; i < kTile; i += kSortThreads) s[i] = i < n ? keys[t0 + i] : ~0ull;
    __syncthreads();
    for (uint32_t size = 2; size <= kTile; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < kTile / 2; i += kSortThreads) {
                const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const unsigned long long a = s[lo], b = s[hi];
                if ((a > b) == up) {
                    s[lo] = b;
                    s[hi] = a;
                }
            }
            __syncthreads();
        }
    for (uint32_t i = threadIdx.x; i < n; i += kSortThreads) keys[t0 + i] = s[i];
}

// number of elements taken from A among the first d outputs of merge(A, B)
__device__ __forceinline__ uint32_t merge_split(const unsigned long long* A, uint32_t na,
                                                const unsigned long long* B, uint32_t nb, uint32_t d) {
    uint32_t lo = d > nb ? d - nb : 0u, hi = min(d, na);
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;  // take mid from A, d - mid from B
        if (A[mid] < B[d - mid - 1])
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(kSortThreads) merge_pass_kernel(const unsigned long long* in,
                                                                  unsigned long long* out,
                                                                  const unsigned long long* count, uint64_t cap,
                                                                  uint32_t width, uint32_t* passes) {
    __shared__ unsigned long long sa[kMTile], sb[kMTile];
    const uint32_t live = live_keys(count, cap);
    if (width >= live) return;  // already one run: nothing to merge (and no pass counted)
    const uint32_t o0 = blockIdx.x * kMTile;
    if (o0 >= live) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(passes, 1u);
    const uint32_t pair = o0 / (2 * width) * (2 * width);
    const uint32_t na = min(width, live - pair), nb = live - pair > width ? min(width, live - pair - width) : 0u;
    const unsigned long long* A = in + pair;
    const unsigned long long* B = A + na;
    const uint32_t d0 = o0 - pair, d1 = min(d0 + kMTile, na + nb);
    __shared__ uint32_t s_split[2];
    if (threadIdx.x < 2) s_split[threadIdx.x] = merge_split(A, na, B, nb, threadIdx.x ? d1 : d0);
    __syncthreads();
    const uint32_t a0 = s_split[0], a1 = s_split[1], b0 = d0 - a0, b1 = d1 - a1;
    const uint32_t ma = a1 - a0, mb = b1 - b0;
    for (uint32_t i = threadIdx.x; i < ma; i += kSortThreads) sa[i] = A[a0 + i];
    for (uint32_t i = threadIdx.x; i < mb; i += kSortThreads) sb[i] = B[b0 + i];
    __syncthreads();
    const uint32_t d = threadIdx.x * kMergePer;
    if (d >= ma + mb) return;
    uint32_t i = merge_split(sa, ma, sb, mb, d), j = d - i;
    const uint32_t e = min(d + kMergePer, ma + mb);
    for (uint32_t o = d; o < e; ++o) {
        const bool takeA = j >= mb || (i < ma && sa[i] < sb[j]);
        out[pair + d0 + o] = takeA ? sa[i++] : sb[j++];
    }
}

// the result is in the scratch buffer after an odd number of effective passes
__global__ void copy_back_kernel(unsigned long long* keys, const unsigned long long* alt,
                                 const unsigned long long* count, uint64_t cap, const uint32_t* passes) {
    if (!(*passes & 1u)) return;
    const uint32_t live = live_keys(count, cap);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < live; i += gridDim.x * blockDim.x) keys[i] = alt[i];
}

// Escape finalisation: keys[0..cap) were pre-filled with ~0 and partially
// overwritten by the kernel's appends; sorting puts the real indices first,
// ascending (the reference's per-shard order).
int sort_escapes(fntrs_ctx* ctx, const EscOut& eout, uint64_t max_key, cudaStream_t st) {
    (void)max_key;
    const uint64_t cap = eout.cap;
    unsigned long long* keys = eout.keys;
    if (cap <= 1) return FNTRS_OK;
    if (cap <= kSmallSort) {
        uint32_t m = 2;
        while (m < cap) m <<= 1;
        const size_t smem = size_t(m) * sizeof(unsigned long long);
        if (smem > 48 * 1024)
            CK(cudaFuncSetAttribute(small_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
               "escape sort attribute");
        small_sort_kernel<<<1, 1024, smem, st>>>(keys, eout.count, uint32_t(cap));
        CK(cudaGetLastError(), "escape sort");
        ctx->launches += 1;
        return FNTRS_OK;
    }
    if (cap > 0x7FFFFFFFull) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "escape capacity too large");
    // per-call, stream-ordered scratch: calls on different streams never share it
    unsigned long long* alt = nullptr;
    CK(cudaMallocAsync(&alt, cap * sizeof(unsigned long long) + 16, st), "escape scratch");
    uint32_t* passes = reinterpret_cast<uint32_t*>(alt + cap);
    CK(cudaMemsetAsync(passes, 0, sizeof(uint32_t), st), "escape sort");
    const uint32_t tiles = uint32_t((cap + kTile - 1) / kTile);
    tile_sort_kernel<<<tiles, kSortThreads, 0, st>>>(keys, eout.count, cap);
    unsigned long long *a = keys, *b = alt;
    int launched = 1;
    const uint32_t mtiles = uint32_t((cap + kMTile - 1) / kMTile);
    for (uint64_t w = kTile; w < cap; w *= 2) {
        merge_pass_kernel<<<mtiles, kSortThreads, 0, st>>>(a, b, eout.count, cap, uint32_t(w), passes);
        std::swap(a, b);
        ++launched;
    }
    // passes the live count did not need exit before writing: the effective ones
    // alternate buffers from `keys`, so an odd count leaves the result in `alt`
    copy_back_kernel<<<148, 256, 0, st>>>(keys, alt, eout.count, cap, passes);
    CK(cudaGetLastError(), "escape sort");
    ctx->launches += launched + 1;
    cudaFreeAsync(alt, st);
    return FNTRS_OK;
}

constexpr size_t kScratchCapDefault = size_t(2) << 30;  // per four-step intermediate buffer
// FNTRS_SCRATCH_MB overrides the four-step batch size (measurement hook)
size_t scratch_cap() {
    static const size_t cap = [] {
        const char* e = getenv("FNTRS_SCRATCH_MB");
        return e ? size_t(atoll(e)) << 20 : kScratchCapDefault;
    }();
    return cap;
}

// Per-call stream-ordered scratch (released in stream order by release_scratch),
// so concurrent calls on different streams never share intermediates.
struct Scratch {
    uint32_t* p[4] = {nullptr, nullptr, nullptr, nullptr};
};
int get_scratch(fntrs_ctx* ctx, Scratch& s, size_t bytes, int count, cudaStream_t st) {
    for (int i = 0; i < count; ++i) CK(cudaMallocAsync(&s.p[i], bytes, st), "scratch alloc");
    return FNTRS_OK;
}
void release_scratch(Scratch& s, cudaStream_t st) {
    for (auto& q : s.p)
        if (q) cudaFreeAsync(q, st);
}

int prep_escapes(fntrs_ctx* ctx, uint64_t* out_esc, uint64_t esc_cap, uint64_t* n_out_esc, cudaStream_t st) {
    if (!n_out_esc) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "n_out_esc must be a device pointer");
    if (esc_cap && !out_esc) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "out_esc is null");
    CK(cudaMemsetAsync(n_out_esc, 0, sizeof(uint64_t), st), "escape count reset");
    if (esc_cap) CK(cudaMemsetAsync(out_esc, 0xFF, esc_cap * sizeof(uint64_t), st), "escape fill");
    return FNTRS_OK;
}

__global__ void negate_scale_kernel(const uint32_t* in, uint32_t* out, uint32_t n, uint32_t s) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = gmul(in[i], s);
}

int encode_impl(fntrs_ctx* ctx, uint32_t k, uint32_t n, uint32_t N, uint32_t stripes, uint32_t L,
                const uint16_t* src, const uint64_t* src_esc, uint64_t n_src_esc, uint16_t* out,
                uint64_t* out_esc, uint64_t esc_cap, uint64_t* n_out_esc, void* stream);

__global__ void set_u64_kernel(uint64_t* p, uint64_t v) { *p = v; }

}  // namespace

extern "C" {

const char* fntrs_gpu_version(void) { return kVersion; }

const char* fntrs_gpu_status_string(int s) {
    switch (s) {
        case FNTRS_OK: return "ok";
        case FNTRS_E_ERROR: return "Error";
        case FNTRS_E_ZERO_INVERSE: return "ZeroInverse";
        case FNTRS_E_INVALID_TRANSFORM_SIZE: return "InvalidTransformSize";
        case FNTRS_E_SIZE_MISMATCH: return "SizeMismatch";
        case FNTRS_E_PRODUCT_TOO_LARGE: return "ProductTooLarge";
        case FNTRS_E_DUPLICATE_POINT: return "DuplicatePoint";
        case FNTRS_E_DUPLICATE_POSITION: return "DuplicatePosition";
        case FNTRS_E_POSITION_OUT_OF_RANGE: return "PositionOutOfRange";
        case FNTRS_E_TOO_FEW_POSITIONS: return "TooFewPositions";
        case FNTRS_E_NOT_ENOUGH_SYMBOLS: return "NotEnoughSymbols";
        case FNTRS_E_TOO_MANY_ESCAPES: return "TooManyEscapes";
        case FNTRS_E_BAD_MAGIC: return "BadMagic";
        case FNTRS_E_BAD_VERSION: return "BadVersion";
        case FNTRS_E_TRUNCATED_SHARD: return "TruncatedShard";
        case FNTRS_E_MALFORMED_ESCAPES: return "MalformedEscapes";
        case FNTRS_E_MALFORMED_HEADER: return "MalformedHeader";
        case FNTRS_E_LENGTH_MISMATCH: return "LengthMismatch";
        case FNTRS_E_NOT_ENOUGH_SHARDS: return "NotEnoughShards";
        case FNTRS_E_CUDA: return "CudaError";
        case FNTRS_E_UNSUPPORTED: return "Unsupported";
        case FNTRS_E_INVALID_ARGUMENT: return "InvalidArgument";
        default: return "unknown";
    }
}

const char* fntrs_gpu_last_error(const fntrs_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }
int fntrs_gpu_device(const fntrs_ctx* ctx) { return ctx ? ctx->device : -1; }
uint64_t fntrs_gpu_launch_count(const fntrs_ctx* ctx) { return ctx ? ctx->launches : 0; }

int fntrs_gpu_transform_counts(const fntrs_ctx* ctx, uint64_t counts[17]) {
    if (!ctx || !counts) return FNTRS_E_INVALID_ARGUMENT;
    std::memcpy(counts, ctx->fnt_counts, sizeof(ctx->fnt_counts));
    return FNTRS_OK;
}

int fntrs_gpu_set_fast_path(fntrs_ctx* ctx, int enabled) {
    if (!ctx) return FNTRS_E_INVALID_ARGUMENT;
    ctx->fast_enabled = enabled != 0;
    return FNTRS_OK;
}

int fntrs_gpu_code_params(uint32_t k, uint32_t n, uint32_t* n_domain) {
    if (k < 1 || k > n || n > 65536) return FNTRS_E_SIZE_MISMATCH;
    if (n_domain) *n_domain = next_pow2(n);
    return FNTRS_OK;
}

int fntrs_gpu_create(int device, fntrs_ctx** out) {
    if (!out) return FNTRS_E_INVALID_ARGUMENT;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count <= 0 || device < 0 || device >= count)
        return FNTRS_E_CUDA;
    auto* ctx = new fntrs_ctx;
    ctx->device = device;
    DeviceGuard g(device);
    cudaError_t e = cudaStreamCreateWithFlags(&ctx->internal, cudaStreamNonBlocking);
    {  // keep stream-ordered allocations (plans, scratch) cached across calls
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t threshold = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
        }
    }
    if (e == cudaSuccess) e = build_tables(ctx->tab, ctx->internal);
    if (e == cudaSuccess) e = fast::build_fast_tables(ctx->ftab, ctx->internal);
    if (e == cudaSuccess) e = fast::upload_const_twiddles(ctx->ftab, ctx->internal);
    if (e == cudaSuccess) e = fast::build_large_tables(ctx->ftab, ctx->internal);
    if (e == cudaSuccess) e = fast::build_log_tables(ctx->ltab, ctx->internal);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->internal);
    if (e != cudaSuccess) {
        delete ctx;
        return FNTRS_E_CUDA;
    }
    ctx->launches = 1;
    *out = ctx;
    return FNTRS_OK;
}

int fntrs_gpu_destroy(fntrs_ctx* ctx) {
    if (!ctx) return FNTRS_OK;
    DeviceGuard g(ctx->device);
    cudaFree(ctx->tab.fwd);
    cudaFree(ctx->tab.inv);
    cudaFree(ctx->ftab.ptab_fwd);
    cudaFree(ctx->ftab.ptab_fwdT);
    cudaFree(ctx->ftab.ptab_inv);
    cudaFree(ctx->ftab.big_fwd);
    cudaFree(ctx->ftab.big_inv);
    cudaFree(ctx->ftab.sys_conv);
    cudaDeviceSynchronize();
    cudaFree(ctx->ltab.exp3);
    cudaFree(ctx->ltab.log3);
    for (auto& kv : ctx->digit_spectra) cudaFree(kv.second);
    // the context's own systematic plans: the device is idle (synchronised
    // above), so free them directly rather than on the stream they were built
    // on, which the caller may already have destroyed
    for (auto& kv : ctx->sys_plans) {
        fntrs_plans* pl = kv.second;
        for (void* p : {(void*)pl->pos, (void*)pl->ainv, (void*)pl->ahat, (void*)pl->rowmap, (void*)pl->ahat2,
                        (void*)pl->alo, (void*)pl->ahi, (void*)pl->sys_w})
            if (p) cudaFree(p);
        delete pl;
    }
    if (ctx->internal) cudaStreamDestroy(ctx->internal);
    delete ctx;
    return FNTRS_OK;
}

int fntrs_gpu_encode(fntrs_ctx* ctx, uint32_t k, uint32_t n, uint32_t stripes, uint32_t L,
                     const uint16_t* src, const uint64_t* src_esc, uint64_t n_src_esc, uint16_t* out,
                     uint64_t* out_esc, uint64_t esc_cap, uint64_t* n_out_esc, void* stream) {
    if (!ctx) return FNTRS_E_INVALID_ARGUMENT;
    uint32_t N = 0;
    if (fntrs_gpu_code_params(k, n, &N))
        return fail(ctx, FNTRS_E_SIZE_MISMATCH, "code parameters need 1 <= k <= n <= 65536, got k = " +
                                                    std::to_string(k) + ", n = " + std::to_string(n));
    return encode_impl(ctx, k, n, N, stripes, L, src, src_esc, n_src_esc, out, out_esc, esc_cap, n_out_esc, stream);
}

}  // extern "C"

namespace {
// FNT_N of k source symbols per codeword, first n outputs (n <= N): the
// kernels behind fntrs_gpu_encode, with the transform size given explicitly.
int encode_impl(fntrs_ctx* ctx, uint32_t k, uint32_t n, uint32_t N, uint32_t stripes, uint32_t L,
                const uint16_t* src, const uint64_t* src_esc, uint64_t n_src_esc, uint16_t* out,
                uint64_t* out_esc, uint64_t esc_cap, uint64_t* n_out_esc, void* stream) {
    const bool large = fast::large_supported(N) && L % fast::large_tile_columns() == 0 && narrow_rows(N, L);
    if (stripes && L && (!src || !out)) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "null buffer");
    if (n_src_esc && !src_esc) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "src_esc is null");
    DeviceGuard g(ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int rc = prep_escapes(ctx, out_esc, esc_cap, n_out_esc, st);
    if (rc) return rc;
    EscIn ein{reinterpret_cast<const unsigned long long*>(src_esc), n_src_esc};
    EscOut eout{reinterpret_cast<unsigned long long*>(out_esc), reinterpret_cast<unsigned long long*>(n_out_esc),
                esc_cap};
    note_fnt(ctx, N, uint64_t(stripes) * L);  // every encode kernel: one FNT_N per codeword
    const int cols = fast::fast_encode_columns(N);
    const bool fast_ok = ctx->fast_enabled && cols && L % uint32_t(cols) == 0 && narrow_rows(N, L) &&
                         reinterpret_cast<uintptr_t>(src) % 16 == 0;
    if (N > kTileMaxN && !large) {  // general column path (codec_cols.cu)
        if (stripes && L) {
            const uint64_t cap = std::min<uint64_t>(uint64_t(stripes) * L, fast::cols_batch_columns(N, kScratchCapDefault));
            Scratch sc;
            rc = get_scratch(ctx, sc, size_t(N) * cap * 4, 2, st);
            if (rc) return rc;
            cudaError_t le = fast::launch_encode_cols(ctx->ftab, k, n, N, stripes, L, src, ein, out, eout, sc.p[0],
                                                      sc.p[1], cap, st);
            release_scratch(sc, st);
            CK(le, "encode launch");
            ctx->launches += 3 * ((uint64_t(stripes) * L + cap - 1) / cap);
        }
        return sort_escapes(ctx, eout, uint64_t(stripes) * n * L, st);
    }
    if (large && fast::stream_enabled()) {
        if (stripes && L) {
            Scratch sc;
            rc = get_scratch(ctx, sc, fast::stream_scratch_words(N, stripes, L, false) * 4, 1, st);
            if (rc) return rc;
            cudaError_t le = fast::launch_encode_stream(ctx->ftab, k, n, N, stripes, L, src, ein, out, eout, sc.p[0], st);
            release_scratch(sc, st);
            CK(le, "encode launch");
            ctx->launches += 1;
        }
        return sort_escapes(ctx, eout, uint64_t(stripes) * n * L, st);
    }
    if (large) {
        if (stripes && L) {
            const uint32_t batch = std::min(stripes, fast::large_batch(N, L, scratch_cap()));
            Scratch sc;
            rc = get_scratch(ctx, sc, size_t(batch) * N * L * 4, 1, st);
            if (rc) return rc;
            cudaError_t le = fast::launch_encode_large(ctx->ftab, k, n, N, stripes, L, src, ein, out, eout, sc.p[0], batch, st);
            release_scratch(sc, st);
            CK(le, "encode launch");
            ctx->launches += 2 * ((stripes + batch - 1) / batch);
        }
        return sort_escapes(ctx, eout, uint64_t(stripes) * n * L, st);
    }
    if (fast_ok)
        CK(fast::launch_encode_fast(ctx->ftab, k, n, N, stripes, L, src, ein, out, eout, st), "encode launch");
    else
        CK(launch_encode_tile(ctx->tab, k, n, N, stripes, L, src, ein, out, eout, st), "encode launch");
    ctx->launches += 1;
    return sort_escapes(ctx, eout, uint64_t(stripes) * n * L, st);
}
}  // namespace

extern "C" {

}  // extern "C"

namespace {
// Plan method for the fused kernels' plans. Direct products cost
// P (k + M) k field multiplies; the log-domain method ~ P N log N (1 + D)
// plus a fixed chain of small launches. FNTRS_PLAN=direct|log overrides.
bool plan_direct(uint32_t k, uint32_t M, uint32_t P) {
    if (const char* m = std::getenv("FNTRS_PLAN")) {
        if (!std::strcmp(m, "direct")) return true;
        if (!std::strcmp(m, "log")) return false;
    }
    // measured (one B200): 1 pattern, k = 1024: direct 0.05 ms vs 0.09 ms; 2049
    // patterns, k = 128 (100M multiplies): a tie; k >= 2048: the log domain by 2.5-10x
    return uint64_t(P) * (uint64_t(k) + M) * k <= (uint64_t(1) << 26);
}
}  // namespace

extern "C" {

int fntrs_gpu_plans_create(fntrs_ctx* ctx, uint32_t k, uint32_t n, uint32_t kp, uint32_t npatterns,
                           const uint32_t* positions, fntrs_plans** out, void* stream) {
    if (!ctx || !out) return FNTRS_E_INVALID_ARGUMENT;
    *out = nullptr;
    uint32_t N = 0;
    if (fntrs_gpu_code_params(k, n, &N))
        return fail(ctx, FNTRS_E_SIZE_MISMATCH, "code parameters need 1 <= k <= n <= 65536");
    const bool full = (kp == n && n == N);  // complete reception: one inverse transform
    if (kp < k) return fail(ctx, FNTRS_E_NOT_ENOUGH_SYMBOLS, "have " + std::to_string(kp) + " symbols, need " + std::to_string(k));
    if (kp != k && !full)
        return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "kp must equal k (or n for complete reception)");
    // 2k > 65536: no product transform fits (interp.cpp:63-67); the product runs by halves
    const bool split = 2ull * k > 65536ull && !full;
    const uint32_t M = split ? 65536u : (2ull * k > 65536ull ? 0u : next_pow2(2 * k));
    // locator data: needed for decoding unless complete; kept for export when it fits
    const bool locator = !full || (kp == k && M && M <= kTileMaxN);
    const bool large = fast::large_supported(N) && !full && !split && kp == k && M == N;
    // shapes neither the fused nor the tile kernels take: the general column path
    const bool cols = split || (!large && (N > kTileMaxN || (!full && M > kTileMaxN)));
    if (npatterns && !positions) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "positions is null");
    // validation (codec.cpp:32-48 order: range first, then duplicates); the
    // duplicate check stamps positions with the pattern number, so nothing is
    // cleared between patterns (O(kp) host work per pattern)
    std::vector<uint32_t> seen(n, 0xFFFFFFFFu);
    for (uint32_t p = 0; p < npatterns; ++p) {
        const uint32_t* z = positions + size_t(p) * kp;
        uint32_t zmax = 0;
        for (uint32_t i = 0; i < kp; ++i) zmax = std::max(zmax, z[i]);
        if (kp && zmax >= n)
            for (uint32_t i = 0; i < kp; ++i)
                if (z[i] >= n)
                    return fail(ctx, FNTRS_E_POSITION_OUT_OF_RANGE, "received position " + std::to_string(z[i]) +
                                                                       " not below n = " + std::to_string(n));
        for (uint32_t i = 0; i < kp; ++i) {
            if (seen[z[i]] == p)
                return fail(ctx, FNTRS_E_DUPLICATE_POSITION, "received position " + std::to_string(z[i]) + " repeats");
            seen[z[i]] = p;
        }
    }
    DeviceGuard g(ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto* pl = new fntrs_plans;
    pl->device = ctx->device;
    pl->k = k;
    pl->n = n;
    pl->N = N;
    pl->M = M;
    pl->kp = kp;
    pl->np = npatterns;
    pl->cols = cols;
    pl->full = full;
    pl->split = split;
    pl->gen = !cols && !full && kp == k && M != N && fast::gen_tile_columns(N, M) != 0;
    pl->ninv = cpow(N % kP, kP - 2);
    const size_t npos = size_t(npatterns) * kp;
    cudaError_t e = cudaSuccess;
    pl->stream = st;
    if (npatterns) {
        e = cudaMallocAsync(&pl->pos, npos * 4, st);
        if (!e) e = cudaMallocAsync(&pl->ainv, npos * 4, st);
        if (!e && locator) e = cudaMallocAsync(&pl->ahat, size_t(npatterns) * M * 4, st);
        if (!e) e = cudaMemcpyAsync(pl->pos, positions, npos * 4, cudaMemcpyHostToDevice, st);
        const bool fastplan = !full && !split && kp == k && M == N && (fast::fast_tile_columns(N) || large);
        if (!e && fastplan && plan_direct(k, M, npatterns)) {
            // few or small patterns: the direct products (plan_build.cu) beat the
            // log-domain method's chain of column transforms
            e = cudaMallocAsync(&pl->rowmap, size_t(npatterns) * N * sizeof(uint2), st);
            if (!e) e = cudaMallocAsync(&pl->ahat2, size_t(npatterns) * N * sizeof(uint2), st);
            if (!e) e = launch_plan_build(N, M, kp, npatterns, pl->pos, pl->ainv, pl->ahat, ctx->tab, st);
            if (!e)
                e = fast::launch_fast_plan_tables(N, kp, npatterns, pl->pos, pl->ainv, pl->ahat, pl->rowmap, pl->ahat2,
                                                  st);
            ctx->launches += 3;
        } else if (!e && fastplan) {
            // log-domain convolution plan (plan_fast.cu): ainv, ahat, rowmap, ahat2 at once
            e = cudaMallocAsync(&pl->rowmap, size_t(npatterns) * N * sizeof(uint2), st);
            if (!e) e = cudaMallocAsync(&pl->ahat2, size_t(npatterns) * N * sizeof(uint2), st);
            const uint32_t w = fast::plan_digit_width(k), D = (16 + w - 1) / w;
            uint32_t* Dh = nullptr;
            auto it = ctx->digit_spectra.find({N, w});
            if (!e && it == ctx->digit_spectra.end()) {
                uint32_t* tmp = nullptr;
                e = cudaMalloc(&Dh, size_t(N) * D * 4);
                if (!e) e = cudaMallocAsync(&tmp, size_t(N) * D * 4 + 256, st);
                if (!e) e = fast::build_digit_spectra(ctx->ftab, ctx->tab, ctx->ltab, N, w, Dh, tmp, st);
                if (tmp) cudaFreeAsync(tmp, st);
                if (!e) ctx->digit_spectra[{N, w}] = Dh;
                ctx->launches += 2;
                note_fnt(ctx, N, D);
            } else if (!e) {
                Dh = it->second;
            }
            uint32_t* scratch = nullptr;
            if (!e) e = cudaMallocAsync(&scratch, fast::plan_fast_scratch_words(N, k, npatterns) * 4, st);
            if (!e)
                e = fast::launch_plan_fast(ctx->ftab, ctx->tab, ctx->ltab, N, k, npatterns, pl->pos, Dh, scratch,
                                           pl->ainv, pl->ahat, pl->rowmap, pl->ahat2, st);
            if (scratch) cudaFreeAsync(scratch, st);
            ctx->launches += 8;
            note_fnt(ctx, N, uint64_t(npatterns) * (1 + D));  // indicator spectra + D digit convolutions
        } else if (!e && locator) {
            e = launch_plan_build(N, M, kp, npatterns, pl->pos, pl->ainv, pl->ahat, ctx->tab, st);
            ctx->launches += 1;
        }
        if (!e && fastplan && N <= kTileMaxN && FNTRS_SYS_CONV_HOST && fast::fast_tile_columns(N)) {
            // output weights of the convolution-form systematic kernels (codec_dec.cu MODE 3 / 4),
            // queued on the plan's stream like rowmap / ahat2 (no synchronisation: capturable)
            e = cudaMallocAsync(&pl->sys_w, size_t(npatterns) * N * sizeof(uint2), st);
            if (!e) e = fast::launch_sys_weights(ctx->ftab, N, npatterns, pl->ahat2, pl->sys_w, st);
            ctx->launches += 1;
        }
        if (!e && pl->gen) {  // fused M != N decode: row map + Shoup pairs of -A_hat/M
            e = cudaMallocAsync(&pl->rowmap, size_t(npatterns) * N * sizeof(uint2), st);
            if (!e) e = cudaMallocAsync(&pl->ahat2, size_t(npatterns) * M * sizeof(uint2), st);
            if (!e) e = fast::build_cols_rowmap(N, kp, npatterns, pl->pos, pl->ainv, pl->rowmap, st);
            if (!e) e = fast::build_gen_pairs(M, npatterns, pl->ahat, pl->ahat2, st);
            ctx->launches += 3;
        }
        if (!e && cols) {  // received-row map for the column path's scatter loader
            e = cudaMallocAsync(&pl->rowmap, size_t(npatterns) * N * sizeof(uint2), st);
            if (!e) e = fast::build_cols_rowmap(N, kp, npatterns, pl->pos, full ? nullptr : pl->ainv, pl->rowmap, st);
            ctx->launches += 2;
        }
        if (!e && split) {  // spectra of the locator's halves (build_split_spectra)
            const size_t words = size_t(M) * npatterns;
            uint32_t *c = nullptr, *T = nullptr;
            e = cudaMallocAsync(&pl->alo, words * 4, st);
            if (!e) e = cudaMallocAsync(&pl->ahi, words * 4, st);
            if (!e) e = cudaMallocAsync(&c, words * 4, st);
            if (!e) e = cudaMallocAsync(&T, words * 4, st);
            if (!e) e = fast::build_split_spectra(ctx->ftab, k, npatterns, pl->ahat, pl->alo, pl->ahi, c, T, st);
            note_fnt(ctx, 65536, 3ull * npatterns);
            if (c) cudaFreeAsync(c, st);
            if (T) cudaFreeAsync(T, st);
            ctx->launches += 6;
        }
    }
    if (e) {
        fntrs_gpu_plans_destroy(pl);
        return cuda_fail(ctx, e, "plan build");
    }
    *out = pl;
    return FNTRS_OK;
}

int fntrs_gpu_plans_destroy(fntrs_plans* pl) {
    if (!pl) return FNTRS_OK;
    DeviceGuard g(pl->device);
    // stream-ordered release: work already queued on the plan's stream may
    // still read the buffers; callers using other streams must order them
    for (void* p : {(void*)pl->pos, (void*)pl->ainv, (void*)pl->ahat, (void*)pl->rowmap, (void*)pl->ahat2,
                    (void*)pl->alo, (void*)pl->ahi, (void*)pl->sys_w})
        if (p) cudaFreeAsync(p, pl->stream);
    delete pl;
    return FNTRS_OK;
}

uint32_t fntrs_gpu_plans_count(const fntrs_plans* pl) { return pl ? pl->np : 0; }

int fntrs_gpu_plans_export(fntrs_ctx* ctx, const fntrs_plans* pl, uint32_t pattern, uint32_t* a_coeffs,
                           uint32_t* aprime_inv, uint32_t* product_size, uint32_t* a_fnt) {
    if (!ctx || !pl) return FNTRS_E_INVALID_ARGUMENT;
    if (pattern >= pl->np) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "pattern out of range");
    if (!pl->ahat) return fail(ctx, FNTRS_E_UNSUPPORTED, "this plan carries no locator (complete reception)");
    DeviceGuard g(ctx->device);
    // the plan was built on the caller's stream; the export runs on the context's own
    CK(cudaDeviceSynchronize(), "export sync");
    cudaStream_t st = ctx->internal;
    const uint32_t M = pl->M, kp = pl->kp;
    uint32_t *acoef = nullptr, *spec = nullptr;
    CK(cudaMalloc(&acoef, M * 4), "export alloc");
    CK(cudaMalloc(&spec, M * 4), "export alloc");
    // A = IFNT_M(A_hat) = -IFNT_unscaled(ahat) since ahat = -A_hat / M
    const uint32_t* ah = pl->ahat + size_t(pattern) * M;
    if (M <= kTileMaxN) {
        CK(launch_fnt_tile(ctx->tab, M, true, kP - 1u, 1, ah, acoef, st), "export ifnt");
        CK(launch_fnt_tile(ctx->tab, M, false, 1u, 1, acoef, spec, st), "export fnt");
    } else {  // A = IFNT_M(-M ahat): scale the inverse by -M * (1/M) = -1 via a forward-then-negate pair
        Scratch sc;
        int rc = get_scratch(ctx, sc, size_t(M) * 4 + 256, 1, st);
        if (rc) return rc;
        CK(fast::launch_fnt_cols(ctx->ftab, M, true, 1, ah, sc.p[0], spec, st), "export ifnt");
        negate_scale_kernel<<<(M + 255) / 256, 256, 0, st>>>(spec, acoef, M, kP - (M % kP));  // * (-M)
        CK(fast::launch_fnt_cols(ctx->ftab, M, false, 1, acoef, sc.p[0], spec, st), "export fnt");
        release_scratch(sc, st);
    }
    ctx->launches += 2;
    std::vector<uint32_t> a(M), sp(M);
    CK(cudaMemcpyAsync(a.data(), acoef, M * 4, cudaMemcpyDeviceToHost, st), "export copy");
    CK(cudaMemcpyAsync(sp.data(), spec, M * 4, cudaMemcpyDeviceToHost, st), "export copy");
    if (aprime_inv)
        CK(cudaMemcpyAsync(aprime_inv, pl->ainv + size_t(pattern) * kp, kp * 4, cudaMemcpyDeviceToHost, st),
           "export copy");
    CK(cudaStreamSynchronize(st), "export sync");
    cudaFree(acoef);
    cudaFree(spec);
    if (a_coeffs) std::memcpy(a_coeffs, a.data(), size_t(kp + 1 <= M ? kp + 1 : M) * 4);
    if (product_size) *product_size = pl->split ? 0u : M;  // interp.cpp:63-67: no product transform
    if (a_fnt && !pl->split) {  // dif_forward leaves the spectrum in bit-reversed order (transform.hpp:43-48)
        int lg = 0;
        while ((1u << lg) < M) ++lg;
        for (uint32_t i = 0; i < M; ++i) {
            uint32_t r = 0;
            for (int b = 0; b < lg; ++b) r |= ((i >> b) & 1u) << (lg - 1 - b);
            a_fnt[i] = sp[r];
        }
    }
    return FNTRS_OK;
}

int fntrs_gpu_decode(fntrs_ctx* ctx, const fntrs_plans* pl, uint32_t stripes, uint32_t L,
                     const uint32_t* stripe_pattern, const uint16_t* rx, const uint64_t* rx_esc,
                     uint64_t n_rx_esc, uint16_t* out, uint64_t* out_esc, uint64_t esc_cap,
                     uint64_t* n_out_esc, void* stream) {
    if (!ctx || !pl) return FNTRS_E_INVALID_ARGUMENT;
    if (pl->device != ctx->device) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "plans belong to another device");
    if (stripes && L && (!rx || !out || !stripe_pattern)) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "null buffer");
    if (stripes && !pl->np) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "no plans");
    if (n_rx_esc && !rx_esc) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "rx_esc is null");
    DeviceGuard g(ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int rc = prep_escapes(ctx, out_esc, esc_cap, n_out_esc, st);
    if (rc) return rc;
    PlanView pv{pl->N, pl->M, pl->kp, pl->k, pl->np, pl->pos, pl->ainv, pl->ahat, pl->ninv};
    EscIn ein{reinterpret_cast<const unsigned long long*>(rx_esc), n_rx_esc};
    EscOut eout{reinterpret_cast<unsigned long long*>(out_esc), reinterpret_cast<unsigned long long*>(n_out_esc),
                esc_cap};
    note_decode_schedule(ctx, pl, uint64_t(stripes) * L);
    const int tcols = fast::fast_tile_columns(pl->N);
    const bool narrow = narrow_rows(std::max(pl->N, pl->M), L);
    const bool fast_ok = ctx->fast_enabled && !pl->cols && !pl->gen && pl->rowmap && tcols && narrow &&
                         L % uint32_t(tcols) == 0 && reinterpret_cast<uintptr_t>(rx) % 16 == 0;
    const int gcols = pl->gen ? fast::gen_tile_columns(pl->N, pl->M) : 0;
    const bool gen_ok = ctx->fast_enabled && gcols && L % uint32_t(gcols) == 0 && narrow &&
                        reinterpret_cast<uintptr_t>(rx) % 16 == 0;
    const bool large_plan = !pl->cols && fast::large_supported(pl->N) && pl->rowmap;
    if (pl->cols || (large_plan && (L % fast::large_tile_columns() || !narrow))) {  // general column path
        if (stripes && L) {
            const uint32_t D = std::max(pl->N, pl->M);
            const uint64_t cap = std::min<uint64_t>(uint64_t(stripes) * L, fast::cols_batch_columns(D, kScratchCapDefault));
            Scratch sc;
            rc = get_scratch(ctx, sc, size_t(D) * cap * 4, pl->split ? 4 : 3, st);
            if (rc) return rc;
            fast::ColsPlanView cv{pl->N,      pl->full ? pl->N : pl->M, pl->k,      pl->kp,  pl->np, pl->full,
                                  pl->split,  pl->rowmap,               pl->ahat,   pl->alo, pl->ahi};
            cudaError_t le = fast::launch_decode_cols(ctx->ftab, cv, stripes, L, stripe_pattern, rx, ein, out, eout,
                                                      sc.p[0], sc.p[1], sc.p[3], sc.p[2], cap, st);
            release_scratch(sc, st);
            CK(le, "decode launch");
            ctx->launches += 7 * ((uint64_t(stripes) * L + cap - 1) / cap);
        }
    } else if (large_plan && fast::stream_enabled()) {
        if (stripes && L) {
            Scratch sc;
            rc = get_scratch(ctx, sc, fast::stream_scratch_words(pl->N, stripes, L, true) * 4, 1, st);
            if (rc) return rc;
            fast::FastPlanView fv{pl->N, pl->k, pl->rowmap, pl->ahat2};
            cudaError_t le = fast::launch_decode_stream(ctx->ftab, fv, stripes, L, stripe_pattern, rx, ein, out, eout,
                                                        sc.p[0], st);
            release_scratch(sc, st);
            CK(le, "decode launch");
            ctx->launches += 1;
        }
    } else if (large_plan) {
        if (stripes && L) {
            const uint32_t batch = std::min(stripes, fast::large_batch(pl->N, L, scratch_cap()));
            Scratch sc;
            rc = get_scratch(ctx, sc, size_t(batch) * pl->N * L * 4, 2, st);
            if (rc) return rc;
            fast::FastPlanView fv{pl->N, pl->k, pl->rowmap, pl->ahat2};
            cudaError_t le = fast::launch_decode_large(ctx->ftab, fv, stripes, L, stripe_pattern, rx, ein, out, eout,
                                                       sc.p[0], sc.p[1], batch, st);
            release_scratch(sc, st);
            CK(le, "decode launch");
            ctx->launches += 4 * ((stripes + batch - 1) / batch);
        }
    } else if (fast_ok) {
        fast::FastPlanView fv{pl->N, pl->k, pl->rowmap, pl->ahat2};
        CK(fast::launch_decode_fast(ctx->ftab, fv, stripes, L, stripe_pattern, rx, ein, out, eout, st), "decode launch");
    } else if (gen_ok) {
        fast::GenPlanView gv{pl->N, pl->M, pl->k, pl->rowmap, pl->ahat2};
        CK(fast::launch_decode_gen(ctx->ftab, gv, stripes, L, stripe_pattern, rx, ein, out, eout, st), "decode launch");
    } else {
        CK(launch_decode_tile(ctx->tab, pv, stripes, L, stripe_pattern, rx, ein, out, eout, st), "decode launch");
    }
    ctx->launches += 1;
    return sort_escapes(ctx, eout, uint64_t(stripes) * pl->k * L, st);
}

}  // extern "C"

namespace {
// The fused systematic kernel serves the plans the fused decode kernel serves
// (n_domain <= 4096, product size == n_domain, L a multiple of its tile width).
bool fused_systematic_ok(const fntrs_ctx* ctx, const fntrs_plans* pl, uint32_t L, const void* in) {
    const int tcols = fast::fast_tile_columns(pl->N);
    return ctx->fast_enabled && narrow_rows(pl->N, L) && pl->rowmap && pl->ahat2 && !pl->cols && !pl->gen && !pl->full && tcols &&
           L % uint32_t(tcols) == 0 && reinterpret_cast<uintptr_t>(in) % 16 == 0;
}

// Interpolation stage of the systematic codec: P = interpolate(plan, rx) into a
// stream-ordered [stripes][k][L] intermediate with its sorted escape list. The
// escape count is read back (one stream synchronisation) so the list can never
// silently overflow; a second pass runs with the exact capacity if it did.
struct Interp {
    uint16_t* coef = nullptr;
    uint64_t* esc = nullptr;
    uint64_t* cnt = nullptr;
    uint64_t n_esc = 0;
    void release(cudaStream_t st) {
        for (void* p : {(void*)coef, (void*)esc, (void*)cnt})
            if (p) cudaFreeAsync(p, st);
    }
};
int interpolate_stage(fntrs_ctx* ctx, const fntrs_plans* pl, uint32_t stripes, uint32_t L, const uint32_t* sp,
                      const uint16_t* rx, const uint64_t* rx_esc, uint64_t n_rx_esc, cudaStream_t st, Interp& it) {
    const uint64_t syms = uint64_t(stripes) * pl->k * L;
    uint64_t cap = syms / 4096 + 4096;
    CK(cudaMallocAsync(&it.coef, std::max<uint64_t>(syms, 1) * 2, st), "systematic intermediate");
    CK(cudaMallocAsync(&it.cnt, sizeof(uint64_t), st), "systematic intermediate");
    for (int attempt = 0; attempt < 2; ++attempt) {
        CK(cudaMallocAsync(&it.esc, cap * sizeof(uint64_t), st), "systematic intermediate");
        int rc = fntrs_gpu_decode(ctx, pl, stripes, L, sp, rx, rx_esc, n_rx_esc, it.coef, it.esc, cap, it.cnt, st);
        if (rc) return rc;
        uint64_t got = 0;
        CK(cudaMemcpyAsync(&got, it.cnt, sizeof(uint64_t), cudaMemcpyDeviceToHost, st), "escape count");
        CK(cudaStreamSynchronize(st), "escape count");
        if (got <= cap) {
            it.n_esc = got;
            return FNTRS_OK;
        }
        cudaFreeAsync(it.esc, st);
        it.esc = nullptr;
        cap = got;
    }
    return fail(ctx, FNTRS_E_TOO_MANY_ESCAPES, "systematic intermediate escape list overflowed");
}
}  // namespace

extern "C" {

int fntrs_gpu_encode_systematic(fntrs_ctx* ctx, uint32_t k, uint32_t n, uint32_t stripes, uint32_t L,
                                const uint16_t* src, const uint64_t* src_esc, uint64_t n_src_esc,
                                uint16_t* out, uint64_t* out_esc, uint64_t esc_cap, uint64_t* n_out_esc,
                                void* stream) {
    if (!ctx) return FNTRS_E_INVALID_ARGUMENT;
    uint32_t N = 0;
    if (fntrs_gpu_code_params(k, n, &N))
        return fail(ctx, FNTRS_E_SIZE_MISMATCH, "code parameters need 1 <= k <= n <= 65536, got k = " +
                                                    std::to_string(k) + ", n = " + std::to_string(n));
    if (stripes && L && (!src || !out)) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "null buffer");
    if (n_src_esc && !src_esc) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "src_esc is null");
    DeviceGuard g(ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (k == n) {  // no parity: the codeword is the source
        int rc = prep_escapes(ctx, out_esc, esc_cap, n_out_esc, st);
        if (rc) return rc;
        const uint64_t bytes = uint64_t(stripes) * k * L * 2;
        if (bytes) CK(cudaMemcpyAsync(out, src, bytes, cudaMemcpyDeviceToDevice, st), "systematic copy");
        const uint64_t keep = std::min(n_src_esc, esc_cap);
        if (keep) CK(cudaMemcpyAsync(out_esc, src_esc, keep * 8, cudaMemcpyDeviceToDevice, st), "systematic copy");
        set_u64_kernel<<<1, 1, 0, st>>>(n_out_esc, n_src_esc);
        CK(cudaGetLastError(), "systematic copy");
        ctx->launches += 1;
        return FNTRS_OK;
    }
    fntrs_plans* pl = nullptr;
    auto found = ctx->sys_plans.find({k, n});
    if (found != ctx->sys_plans.end()) {
        pl = found->second;
    } else {
        std::vector<uint32_t> pos(k);
        for (uint32_t i = 0; i < k; ++i) pos[i] = i;
        int rc = fntrs_gpu_plans_create(ctx, k, n, k, 1, pos.data(), &pl, stream);
        if (rc) return rc;
        CK(cudaStreamSynchronize(st), "systematic plan");  // later calls may use other streams
        ctx->sys_plans[{k, n}] = pl;
    }
    if (!stripes || !L) {
        int rc = prep_escapes(ctx, out_esc, esc_cap, n_out_esc, st);
        return rc;
    }
    uint32_t* sp = nullptr;
    CK(cudaMallocAsync(&sp, size_t(stripes) * 4, st), "systematic pattern map");
    CK(cudaMemsetAsync(sp, 0, size_t(stripes) * 4, st), "systematic pattern map");
    if (fused_systematic_ok(ctx, pl, L, src)) {  // one kernel: interpolate, re-encode, copy the source rows
        int rc = prep_escapes(ctx, out_esc, esc_cap, n_out_esc, st);
        if (!rc) {
            EscIn ein{reinterpret_cast<const unsigned long long*>(src_esc), n_src_esc};
            EscOut eout{reinterpret_cast<unsigned long long*>(out_esc), reinterpret_cast<unsigned long long*>(n_out_esc),
                        esc_cap};
            fast::FastPlanView fv{pl->N, pl->k, pl->rowmap, pl->ahat2, pl->sys_w};
            note_fnt(ctx, pl->N, (pl->sys_w ? 2ull : 4ull) * stripes * L);  // conv form: 2 transforms; else 3 + 1
            cudaError_t le = fast::launch_systematic_fast(ctx->ftab, fv, true, n, stripes, L, sp, src, ein, out, eout, st);
            cudaFreeAsync(sp, st);
            CK(le, "systematic encode launch");
            ctx->launches += 1;
            rc = sort_escapes(ctx, eout, uint64_t(stripes) * n * L, st);
        }
        return rc;
    }
    Interp it;
    int rc = interpolate_stage(ctx, pl, stripes, L, sp, src, src_esc, n_src_esc, st, it);
    if (!rc) rc = encode_impl(ctx, k, n, N, stripes, L, it.coef, it.esc, it.n_esc, out, out_esc, esc_cap, n_out_esc, stream);
    it.release(st);
    cudaFreeAsync(sp, st);
    return rc;
}

int fntrs_gpu_decode_systematic(fntrs_ctx* ctx, const fntrs_plans* pl, uint32_t stripes, uint32_t L,
                                const uint32_t* stripe_pattern, const uint16_t* rx, const uint64_t* rx_esc,
                                uint64_t n_rx_esc, uint16_t* out, uint64_t* out_esc, uint64_t esc_cap,
                                uint64_t* n_out_esc, void* stream) {
    if (!ctx || !pl) return FNTRS_E_INVALID_ARGUMENT;
    if (pl->device != ctx->device) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "plans belong to another device");
    if (stripes && L && (!rx || !out || !stripe_pattern)) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "null buffer");
    if (stripes && !pl->np) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "no plans");
    if (n_rx_esc && !rx_esc) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "rx_esc is null");
    DeviceGuard g(ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (!stripes || !L) return prep_escapes(ctx, out_esc, esc_cap, n_out_esc, st);
    if (fused_systematic_ok(ctx, pl, L, rx)) {  // one kernel: interpolate, re-encode rows 0..k-1
        int rc = prep_escapes(ctx, out_esc, esc_cap, n_out_esc, st);
        if (rc) return rc;
        EscIn ein{reinterpret_cast<const unsigned long long*>(rx_esc), n_rx_esc};
        EscOut eout{reinterpret_cast<unsigned long long*>(out_esc), reinterpret_cast<unsigned long long*>(n_out_esc),
                    esc_cap};
        fast::FastPlanView fv{pl->N, pl->k, pl->rowmap, pl->ahat2, pl->sys_w};
        note_fnt(ctx, pl->N, (pl->sys_w ? 2ull : 4ull) * stripes * L);
        CK(fast::launch_systematic_fast(ctx->ftab, fv, false, pl->n, stripes, L, stripe_pattern, rx, ein, out, eout, st),
           "systematic decode launch");
        ctx->launches += 1;
        return sort_escapes(ctx, eout, uint64_t(stripes) * pl->k * L, st);
    }
    Interp it;
    int rc = interpolate_stage(ctx, pl, stripes, L, stripe_pattern, rx, rx_esc, n_rx_esc, st, it);
    if (!rc)
        rc = encode_impl(ctx, pl->k, pl->k, pl->N, stripes, L, it.coef, it.esc, it.n_esc, out, out_esc, esc_cap,
                         n_out_esc, stream);
    it.release(st);
    return rc;
}

int fntrs_gpu_symbolize(fntrs_ctx* ctx, const uint8_t* data, uint64_t len, uint32_t k, uint32_t L, uint16_t* src,
                        void* stream) {
    if (!ctx) return FNTRS_E_INVALID_ARGUMENT;
    if (k == 0) return fail(ctx, FNTRS_E_SIZE_MISMATCH, "symbolize needs k >= 1");
    if ((len + 1) / 2 > uint64_t(k) * L) return fail(ctx, FNTRS_E_LENGTH_MISMATCH, "L too small for the data");
    if ((len && !data) || (L && !src)) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "null buffer");
    DeviceGuard g(ctx->device);
    CK(launch_symbolize(data, len, k, L, src, static_cast<cudaStream_t>(stream)), "symbolize");
    ctx->launches += 1;
    return FNTRS_OK;
}

int fntrs_gpu_desymbolize(fntrs_ctx* ctx, const uint16_t* dec, uint32_t k, uint32_t L, uint64_t len, uint8_t* out,
                          void* stream) {
    if (!ctx) return FNTRS_E_INVALID_ARGUMENT;
    if (k == 0 || len > uint64_t(k) * L * 2) return fail(ctx, FNTRS_E_LENGTH_MISMATCH, "length exceeds capacity");
    if (len && (!dec || !out)) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "null buffer");
    DeviceGuard g(ctx->device);
    CK(launch_desymbolize(dec, k, L, len, out, static_cast<cudaStream_t>(stream)), "desymbolize");
    ctx->launches += 1;
    return FNTRS_OK;
}

int fntrs_gpu_words_to_be(fntrs_ctx* ctx, const uint16_t* rows, uint32_t nrows, uint32_t L, uint32_t count,
                          uint8_t* out, uint64_t pitch, void* stream) {
    if (!ctx) return FNTRS_E_INVALID_ARGUMENT;
    if (count > L || pitch < 2ull * count) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "count/pitch out of range");
    if (nrows && count && (!rows || !out)) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "null buffer");
    DeviceGuard g(ctx->device);
    CK(launch_words_to_be(rows, nrows, L, count, out, pitch, static_cast<cudaStream_t>(stream)), "words_to_be");
    ctx->launches += 1;
    return FNTRS_OK;
}

int fntrs_gpu_be_to_words(fntrs_ctx* ctx, const uint8_t* in, uint64_t pitch, uint32_t nrows, uint32_t count,
                          uint32_t L, uint16_t* rows, void* stream) {
    if (!ctx) return FNTRS_E_INVALID_ARGUMENT;
    if (count > L || pitch < 2ull * count) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "count/pitch out of range");
    if (nrows && L && (!rows || (count && !in))) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "null buffer");
    DeviceGuard g(ctx->device);
    CK(launch_be_to_words(in, pitch, nrows, count, L, rows, static_cast<cudaStream_t>(stream)), "be_to_words");
    ctx->launches += 1;
    return FNTRS_OK;
}

int fntrs_gpu_fnt(fntrs_ctx* ctx, uint32_t m, int inverse, uint32_t L, const uint32_t* in, uint32_t* out,
                  void* stream) {
    if (!ctx) return FNTRS_E_INVALID_ARGUMENT;
    if (m == 0 || m > 65536 || (m & (m - 1)))
        return fail(ctx, FNTRS_E_INVALID_TRANSFORM_SIZE, "transform size must be a power of two in [1, 65536]");
    if (L && (!in || !out)) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "null buffer");
    DeviceGuard g(ctx->device);
    note_fnt(ctx, m, L);
    if (m > kTileMaxN) {  // column-batched four-step kernels (plan_fast.cu)
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        Scratch sc;
        int rc = get_scratch(ctx, sc, size_t(m) * L * 4 + 256, 1, st);
        if (rc) return rc;
        cudaError_t le = fast::launch_fnt_cols(ctx->ftab, m, inverse != 0, L, in, sc.p[0], out, st, inverse == 2);
        release_scratch(sc, st);
        CK(le, "fnt launch");
        ctx->launches += 2;
        return FNTRS_OK;
    }
    const uint32_t scale = inverse == 1 ? cpow(m % kP, kP - 2) : 1u;  // 2: unscaled inverse
    CK(launch_fnt_tile(ctx->tab, m, inverse != 0, scale, L, in, out, static_cast<cudaStream_t>(stream)), "fnt launch");
    ctx->launches += 1;
    return FNTRS_OK;
}

}  // extern "C"

namespace {
__global__ void fill_symbols_kernel(uint64_t seed, uint64_t first, uint64_t count, uint16_t* out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t z = seed + (first + i + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        out[i] = uint16_t(z);
    }
}
}  // namespace

extern "C" int fntrs_gpu_fill_symbols(uint64_t seed, uint64_t first_index, uint64_t count, uint16_t* out,
                                      void* stream) {
    if (!count) return FNTRS_OK;
    if (!out) return FNTRS_E_INVALID_ARGUMENT;
    fill_symbols_kernel<<<148 * 16, 256, 0, static_cast<cudaStream_t>(stream)>>>(seed, first_index, count, out);
    return cudaGetLastError() == cudaSuccess ? FNTRS_OK : FNTRS_E_CUDA;
}

namespace {
void note_decode_schedule(fntrs_ctx* ctx, const fntrs_plans* pl, uint64_t codewords) {
    if (!codewords) return;
    if (pl->full) {
        note_fnt(ctx, pl->N, codewords);
        return;
    }
    note_fnt(ctx, pl->N, codewords);
    if (pl->split) note_fnt(ctx, 65536, 4 * codewords);
    else note_fnt(ctx, pl->M, 2 * codewords);
}
}  // namespace

// ---- the rest of the reference's public API (poly_aux.cu) -------------------
extern "C" {

int fntrs_gpu_naive_dft(fntrs_ctx* ctx, uint32_t root, int inverse, uint32_t n, const uint32_t* in, uint32_t* out,
                        void* stream) {
    if (!ctx) return FNTRS_E_INVALID_ARGUMENT;
    if (n && (!in || !out)) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "null buffer");
    DeviceGuard g(ctx->device);
    root %= kP;
    const uint32_t r = inverse ? cpow(root, kP - 2) : root;                  // gf::inv (field.hpp:47-50)
    const uint32_t scale = inverse ? cpow(uint32_t(n % kP), kP - 2) : 1u;  // inv(n mod p)
    CK(launch_naive_dft(r, scale, n, in, out, static_cast<cudaStream_t>(stream)), "naive dft");
    ctx->launches += 1;
    return FNTRS_OK;
}

int fntrs_gpu_transform_tables(fntrs_ctx* ctx, uint32_t n, uint32_t* twiddles, uint32_t* inverse_twiddles,
                               uint32_t* bit_reversal, uint32_t* stage_twiddles, uint32_t* stage_inverse_twiddles,
                               void* stream) {
    if (!ctx) return FNTRS_E_INVALID_ARGUMENT;
    if (n == 0 || n > 65536 || (n & (n - 1)))
        return fail(ctx, FNTRS_E_INVALID_TRANSFORM_SIZE, "transform size must be a power of two in [1, 65536]");
    DeviceGuard g(ctx->device);
    CK(launch_transform_tables(n, croot(n, false), croot(n, true), twiddles, inverse_twiddles, bit_reversal,
                               stage_twiddles, stage_inverse_twiddles, static_cast<cudaStream_t>(stream)),
       "transform tables");
    ctx->launches += 1;
    return FNTRS_OK;
}

int fntrs_gpu_poly_products(fntrs_ctx* ctx, uint32_t npairs, const fntrs_poly_pair* pairs, const uint32_t* in,
                            uint32_t* out, void* stream) {
    if (!ctx) return FNTRS_E_INVALID_ARGUMENT;
    if (npairs && (!pairs || !in || !out)) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "null buffer");
    DeviceGuard g(ctx->device);
    CK(launch_pair_products(npairs, pairs, in, out, static_cast<cudaStream_t>(stream)), "poly products");
    ctx->launches += 1;
    return FNTRS_OK;
}

int fntrs_gpu_subproduct_tree_layout(uint32_t k, uint32_t* n_levels, uint32_t* level_nodes, uint32_t level_cap,
                                     uint32_t* node_len, uint64_t* n_nodes, uint64_t* n_coeffs) {
    if (k == 0) return FNTRS_E_SIZE_MISMATCH;
    std::vector<uint32_t> lvl;
    const std::vector<uint32_t> len = tree_node_lengths(k, &lvl);
    if (n_levels) *n_levels = uint32_t(lvl.size());
    if (level_nodes) {
        if (level_cap < lvl.size()) return FNTRS_E_INVALID_ARGUMENT;
        std::copy(lvl.begin(), lvl.end(), level_nodes);
    }
    if (node_len) std::copy(len.begin(), len.end(), node_len);
    if (n_nodes) *n_nodes = len.size();
    if (n_coeffs) {
        uint64_t t = 0;
        for (uint32_t l : len) t += l;
        *n_coeffs = t;
    }
    return FNTRS_OK;
}

int fntrs_gpu_subproduct_tree(fntrs_ctx* ctx, uint32_t k, const uint32_t* points, uint32_t* coeffs, void* stream) {
    if (!ctx) return FNTRS_E_INVALID_ARGUMENT;
    if (k == 0) return fail(ctx, FNTRS_E_SIZE_MISMATCH, "subproduct tree needs at least one point");
    if (!points || !coeffs) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "null buffer");
    DeviceGuard g(ctx->device);
    CK(launch_subproduct_tree(k, points, coeffs, static_cast<cudaStream_t>(stream)), "subproduct tree");
    ctx->launches += 2;
    return FNTRS_OK;
}

int fntrs_gpu_lagrange(fntrs_ctx* ctx, uint32_t k, const uint32_t* xs, const uint32_t* vs, uint32_t* out,
                       void* stream) {
    if (!ctx) return FNTRS_E_INVALID_ARGUMENT;
    if (k && (!xs || !vs || !out)) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "null buffer");
    DeviceGuard g(ctx->device);
    CK(launch_lagrange(k, xs, vs, out, static_cast<cudaStream_t>(stream)), "lagrange");
    ctx->launches += 3;
    return FNTRS_OK;
}

int fntrs_gpu_chirp_table(fntrs_ctx* ctx, uint32_t n, uint32_t root, uint32_t* b, uint32_t* b_inverse,
                          uint32_t* b_spectrum, void* stream) {  // geom.cpp:13-41
    if (!ctx) return FNTRS_E_INVALID_ARGUMENT;
    if (n == 0 || n > 65536 || (n & (n - 1)))
        return fail(ctx, FNTRS_E_INVALID_TRANSFORM_SIZE, "chirp table size must be a power of two in [1, 65536]");
    if (n == 65536) return FNTRS_OK;  // full domain: evaluation is the transform itself
    DeviceGuard g(ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch sc;
    int rc = get_scratch(ctx, sc, size_t(4) * n * 4 + 256, 1, st);
    if (rc) return rc;
    uint32_t* bb = b ? b : sc.p[0];
    cudaError_t e = launch_chirp(n, root, bb, b_inverse, st);
    ctx->launches += 1;
    if (!e && b_spectrum) {  // b zero-padded to 2n, forward spectrum
        uint32_t* pad = sc.p[0] + 2 * n;
        e = cudaMemsetAsync(pad, 0, size_t(2) * n * 4, st);
        if (!e) e = cudaMemcpyAsync(pad, bb, size_t(2 * n - 1) * 4, cudaMemcpyDeviceToDevice, st);
        if (!e) rc = fntrs_gpu_fnt(ctx, 2 * n, 0, 1, pad, b_spectrum, stream);
    }
    release_scratch(sc, st);
    if (rc) return rc;
    CK(e, "chirp table");
    return FNTRS_OK;
}

int fntrs_gpu_geom_eval(fntrs_ctx* ctx, uint32_t n, uint32_t root, const uint32_t* a, uint32_t len,
                        const uint32_t* b_inverse, const uint32_t* b_spectrum, uint32_t* out,
                        void* stream) {  // geom.cpp:59-99
    if (!ctx) return FNTRS_E_INVALID_ARGUMENT;
    if (n == 0 || n > 65536 || (n & (n - 1)))
        return fail(ctx, FNTRS_E_INVALID_TRANSFORM_SIZE, "chirp table size must be a power of two in [1, 65536]");
    if (len > n) return fail(ctx, FNTRS_E_SIZE_MISMATCH, "geom_eval: polynomial has more coefficients than points");
    if (!out || (len && !a)) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "null buffer");
    DeviceGuard g(ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    root %= kP;
    Scratch sc;
    int rc = get_scratch(ctx, sc, size_t(8) * n * 4 + 256, 1, st);
    if (rc) return rc;
    cudaError_t e = cudaSuccess;
    if (n == 65536) {  // eval_full_domain: the transform (forward), or its unscaled inverse for the inverse root
        const bool fwd = root == croot(n, false), inv = root == croot(n, true);
        if (!fwd && !inv) {
            release_scratch(sc, st);
            return fail(ctx, FNTRS_E_INVALID_TRANSFORM_SIZE, "full-domain evaluation needs the transform root");
        }
        uint32_t* pad = sc.p[0];
        e = cudaMemsetAsync(pad, 0, size_t(n) * 4, st);
        if (!e && len) e = cudaMemcpyAsync(pad, a, size_t(len) * 4, cudaMemcpyDeviceToDevice, st);
        // sum a_j root^-(ij) = n * fnt_inverse = -fnt_inverse (65536 = -1): the unscaled inverse
        if (!e) rc = fntrs_gpu_fnt(ctx, n, fwd ? 0 : 2, 1, pad, out, stream);
    } else {
        const uint32_t m = 2 * n;
        uint32_t *binv = sc.p[0], *B = binv + n, *c = B + m, *c2 = c + m;
        if (b_inverse && b_spectrum) {  // the caller's cached table
            binv = const_cast<uint32_t*>(b_inverse);
            B = const_cast<uint32_t*>(b_spectrum);
        } else {
            e = launch_chirp(n, root, c2, binv, st);  // b into c2 (2n - 1), then its padded spectrum
            if (!e) e = cudaMemsetAsync(c2 + (m - 1), 0, 4, st);
            if (!e) rc = fntrs_gpu_fnt(ctx, m, 0, 1, c2, B, stream);
        }
        if (!e && !rc) e = launch_geom_pre(n, len, a, binv, c, st);
        if (!e && !rc) rc = fntrs_gpu_fnt(ctx, m, 0, 1, c, c2, stream);
        if (!e && !rc) e = launch_pointwise(m, c2, B, st);
        if (!e && !rc) rc = fntrs_gpu_fnt(ctx, m, 1, 1, c2, c, stream);  // inverse, 1/m
        if (!e && !rc) e = launch_geom_post(n, c, binv, out, st);
        ctx->launches += 4;
    }
    release_scratch(sc, st);
    if (rc) return rc;
    CK(e, "geom eval");
    return FNTRS_OK;
}

int fntrs_gpu_geom_eval_negative(fntrs_ctx* ctx, uint32_t n, uint32_t root, const uint32_t* a, uint32_t len,
                                 const uint32_t* b_inverse, const uint32_t* b_spectrum, uint32_t* out,
                                 void* stream) {  // geom.cpp:101-116
    if (!ctx) return FNTRS_E_INVALID_ARGUMENT;
    if (len > n)
        return fail(ctx, FNTRS_E_SIZE_MISMATCH, "geom_eval_negative: polynomial has more coefficients than points");
    if (!out || (len && !a)) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "null buffer");
    DeviceGuard g(ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint32_t rho = cpow(root % kP, kP - 2);
    Scratch sc;
    int rc = get_scratch(ctx, sc, size_t(len) * 4 + 256, 1, st);
    if (rc) return rc;
    cudaError_t e = launch_powers_scale(len, rho, a, sc.p[0], st);
    ctx->launches += 1;
    if (!e) rc = fntrs_gpu_geom_eval(ctx, n, rho, sc.p[0], len, b_inverse, b_spectrum, out, stream);
    release_scratch(sc, st);
    if (rc) return rc;
    CK(e, "geom eval negative");
    return FNTRS_OK;
}

int fntrs_gpu_poly_derivative(fntrs_ctx* ctx, uint32_t len, const uint32_t* a, uint32_t* out, void* stream) {
    if (!ctx) return FNTRS_E_INVALID_ARGUMENT;
    if (len > 1 && (!a || !out)) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "null buffer");
    DeviceGuard g(ctx->device);
    CK(launch_derivative(len, a, out, static_cast<cudaStream_t>(stream)), "derivative");
    ctx->launches += 1;
    return FNTRS_OK;
}

int fntrs_gpu_poly_eval(fntrs_ctx* ctx, uint32_t len, const uint32_t* a, uint32_t x, uint32_t* out, void* stream) {
    if (!ctx) return FNTRS_E_INVALID_ARGUMENT;
    if (!out || (len && !a)) return fail(ctx, FNTRS_E_INVALID_ARGUMENT, "null buffer");
    DeviceGuard g(ctx->device);
    CK(launch_eval(len, x, a, out, static_cast<cudaStream_t>(stream)), "eval");
    ctx->launches += 1;
    return FNTRS_OK;
}

}  // extern "C"
