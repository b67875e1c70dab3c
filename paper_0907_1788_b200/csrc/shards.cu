// shards.cu -- the shard wire format's data movement on the GPU
// (proj/src/shardio.cpp): file bytes <-> source symbols, and packet rows <->
// big-endian shard payloads. Headers, escape lists and manifests are a few
// bytes per shard and are formatted on the host (paper_0907_1788_b200/shards.py).
//
// Layout: the reference CLI codes a file as S = ceil(words / k) stripes of one
// codeword each (shardio::symbolize, shardio.cpp:83-96: word t*k + i is symbol
// i of stripe t) and shard j carries symbol j of every stripe
// (fntrs_main.cpp:141-149). In the batched model that is ONE stripe whose
// packets are k rows of L >= S symbols: packet i = (word t*k + i for t < S),
// encoded row j = shard j's payload. Symbolize is therefore a transpose of the
// [S][k] word matrix; it runs through 32 x 32 shared tiles so both the byte
// reads and the packet writes are coalesced.
#include <cuda_runtime.h>

#include <cstdint>

namespace fntrs_gpu {
namespace {

constexpr int kT = 32;

// src[i][t] = word(t*k + i) (big-endian byte pair, zero past the data), t < L
__global__ void symbolize_kernel(const uint8_t* __restrict__ data, uint64_t len, uint32_t k, uint32_t L,
                                 uint16_t* __restrict__ src) {
    __shared__ uint16_t tile[kT][kT + 1];
    const uint32_t i0 = blockIdx.x * kT, t0 = blockIdx.y * kT;
    const uint64_t words = (len + 1) / 2;
    // read: row t, consecutive i (contiguous words)
    for (uint32_t r = threadIdx.y; r < kT; r += blockDim.y) {
        const uint32_t t = t0 + r, i = i0 + threadIdx.x;
        uint16_t v = 0;
        if (i < k && t < L) {
            const uint64_t w = uint64_t(t) * k + i;
            if (w < words) {
                const uint32_t hi = data[2 * w];
                const uint32_t lo = 2 * w + 1 < len ? data[2 * w + 1] : 0u;
                v = uint16_t((hi << 8) | lo);
            }
        }
        tile[r][threadIdx.x] = v;
    }
    __syncthreads();
    // write: packet i, consecutive t
    for (uint32_t r = threadIdx.y; r < kT; r += blockDim.y) {
        const uint32_t i = i0 + r, t = t0 + threadIdx.x;
        if (i < k && t < L) src[uint64_t(i) * L + t] = tile[threadIdx.x][r];
    }
}

// out[2w], out[2w+1] = big-endian word w = dec[w % k][w / k], w < ceil(len/2), truncated to len
__global__ void desymbolize_kernel(const uint16_t* __restrict__ dec, uint32_t k, uint32_t L, uint64_t len,
                                   uint8_t* __restrict__ out) {
    __shared__ uint16_t tile[kT][kT + 1];
    const uint32_t i0 = blockIdx.x * kT, t0 = blockIdx.y * kT;
    for (uint32_t r = threadIdx.y; r < kT; r += blockDim.y) {  // read packet i, consecutive t
        const uint32_t i = i0 + r, t = t0 + threadIdx.x;
        tile[r][threadIdx.x] = (i < k && t < L) ? dec[uint64_t(i) * L + t] : uint16_t(0);
    }
    __syncthreads();
    for (uint32_t r = threadIdx.y; r < kT; r += blockDim.y) {  // write row t, consecutive i
        const uint32_t t = t0 + r, i = i0 + threadIdx.x;
        if (i >= k || t >= L) continue;
        const uint64_t w = uint64_t(t) * k + i;
        const uint16_t v = tile[threadIdx.x][r];
        if (2 * w < len) out[2 * w] = uint8_t(v >> 8);
        if (2 * w + 1 < len) out[2 * w + 1] = uint8_t(v);
    }
}

// payload bytes: out[r * pitch + 2t..] = big-endian rows[r][t], t < count
__global__ void words_to_be_kernel(const uint16_t* __restrict__ rows, uint32_t nrows, uint32_t L, uint32_t count,
                                   uint8_t* __restrict__ out, uint64_t pitch) {
    const uint64_t total = uint64_t(nrows) * count;
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < total; j += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t r = uint32_t(j / count), t = uint32_t(j - uint64_t(r) * count);
        const uint16_t v = rows[uint64_t(r) * L + t];
        uint8_t* o = out + uint64_t(r) * pitch + 2ull * t;
        o[0] = uint8_t(v >> 8);
        o[1] = uint8_t(v);
    }
}

// inverse: rows[r][t] = big-endian in[r * pitch + 2t..] for t < count, 0 for count <= t < L
__global__ void be_to_words_kernel(const uint8_t* __restrict__ in, uint64_t pitch, uint32_t nrows, uint32_t count,
                                   uint32_t L, uint16_t* __restrict__ rows) {
    const uint64_t total = uint64_t(nrows) * L;
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < total; j += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t r = uint32_t(j / L), t = uint32_t(j - uint64_t(r) * L);
        uint16_t v = 0;
        if (t < count) {
            const uint8_t* p = in + uint64_t(r) * pitch + 2ull * t;
            v = uint16_t((uint32_t(p[0]) << 8) | p[1]);
        }
        rows[j] = v;
    }
}

}  // namespace

cudaError_t launch_symbolize(const uint8_t* data, uint64_t len, uint32_t k, uint32_t L, uint16_t* src,
                             cudaStream_t st) {
    if (!k || !L) return cudaSuccess;
    const dim3 grid((k + kT - 1) / kT, (L + kT - 1) / kT), block(kT, 8);
    if (grid.y > 65535) return cudaErrorInvalidConfiguration;
    symbolize_kernel<<<grid, block, 0, st>>>(data, len, k, L, src);
    return cudaGetLastError();
}

cudaError_t launch_desymbolize(const uint16_t* dec, uint32_t k, uint32_t L, uint64_t len, uint8_t* out,
                               cudaStream_t st) {
    if (!k || !L || !len) return cudaSuccess;
    const dim3 grid((k + kT - 1) / kT, (L + kT - 1) / kT), block(kT, 8);
    if (grid.y > 65535) return cudaErrorInvalidConfiguration;
    desymbolize_kernel<<<grid, block, 0, st>>>(dec, k, L, len, out);
    return cudaGetLastError();
}

cudaError_t launch_words_to_be(const uint16_t* rows, uint32_t nrows, uint32_t L, uint32_t count, uint8_t* out,
                               uint64_t pitch, cudaStream_t st) {
    if (!nrows || !count) return cudaSuccess;
    words_to_be_kernel<<<148 * 8, 256, 0, st>>>(rows, nrows, L, count, out, pitch);
    return cudaGetLastError();
}

cudaError_t launch_be_to_words(const uint8_t* in, uint64_t pitch, uint32_t nrows, uint32_t count, uint32_t L,
                               uint16_t* rows, cudaStream_t st) {
    if (!nrows || !L) return cudaSuccess;
    be_to_words_kernel<<<148 * 8, 256, 0, st>>>(in, pitch, nrows, count, L, rows);
    return cudaGetLastError();
}

}  // namespace fntrs_gpu
