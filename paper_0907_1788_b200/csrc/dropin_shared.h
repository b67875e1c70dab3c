// dropin_shared.h -- the drop-in API's shared device context (one per
// process, serialised by a mutex: the C ABI requires serialised calls per
// context), its scratch and plan LRU, and the Fe <-> uint16 + escape
// marshalling used by dropin.cpp and dropin_aux.cpp.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <list>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "fntrs/errors.hpp"
#include "fntrs/field.hpp"
#include "fntrs/instrument.hpp"
#include "fntrs/poly.hpp"
#include "fntrs_gpu.h"

namespace fntrs {

void throw_status(int status, const std::string& msg);

namespace dropin {

// One shared context + scratch for the per-codeword API; calls serialise on
// its mutex (the C ABI requires serialised calls per context).
struct Shared {
    std::mutex mu;
    int device = 0;
    fntrs_ctx* ctx = nullptr;
    cudaStream_t stream = nullptr;
    // device scratch
    void* dbuf = nullptr;
    size_t dbuf_bytes = 0;
    uint32_t* zero_pattern = nullptr;  // stripe_pattern of a one-stripe call: {0}
    // plan LRU (interp.cpp:70-101): key (n, k, kp, positions)
    using Key = std::pair<std::vector<uint32_t>, std::vector<uint32_t>>;
    std::list<std::pair<Key, fntrs_plans*>> lru;
    static constexpr size_t kCapacity = 16;
    uint64_t seen[17] = {};  // the context's transform tally already reported to FntScopes

    // Report the transforms the library's kernels executed since the last
    // call (fntrs_gpu_transform_counts) to the calling thread's FntScopes, as
    // the reference's transform layer does per executed transform
    // (transform.cpp:292-316 -> note_fnt_execution).
    void note_transforms() {
        uint64_t now[17];
        if (!ctx || fntrs_gpu_transform_counts(ctx, now)) return;
        for (int e = 0; e < 17; ++e) {
            for (uint64_t i = seen[e]; i < now[e]; ++i) note_fnt_execution(std::size_t{1} << e);
            seen[e] = now[e];
        }
    }

    ~Shared() {
        for (auto& e : lru) fntrs_gpu_plans_destroy(e.second);
        if (dbuf) cudaFree(dbuf);
        if (zero_pattern) cudaFree(zero_pattern);
        if (stream) cudaStreamDestroy(stream);
        if (ctx) fntrs_gpu_destroy(ctx);
    }

    void check(int status) {
        if (status) throw_status(status, std::string(fntrs_gpu_status_string(status)) + ": " +
                                             fntrs_gpu_last_error(ctx));
    }

    void ensure() {
        if (ctx) return;
        int rc = fntrs_gpu_create(device, &ctx);
        if (rc) {
            ctx = nullptr;
            throw Error("fntrs: no usable CUDA device " + std::to_string(device) +
                        " (the codec has no CPU fallback)");
        }
        cudaSetDevice(device);
        if (cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking) != cudaSuccess)
            throw Error("fntrs: cannot create a CUDA stream");
        if (cudaMalloc(&zero_pattern, 4) != cudaSuccess || cudaMemset(zero_pattern, 0, 4) != cudaSuccess)
            throw Error("fntrs: device allocation failed");
    }

    void* scratch(size_t bytes) {
        if (bytes > dbuf_bytes) {
            if (dbuf) cudaFree(dbuf);
            dbuf = nullptr;
            if (cudaMalloc(&dbuf, bytes) != cudaSuccess) throw Error("fntrs: device allocation failed");
            dbuf_bytes = bytes;
        }
        return dbuf;
    }

    void sync() {
        cudaError_t e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) throw Error(std::string("fntrs: CUDA error: ") + cudaGetErrorString(e));
    }

    fntrs_plans* plan_for(uint32_t k, uint32_t n, const std::vector<uint32_t>& pos) {
        Key key{{n, k, uint32_t(pos.size())}, pos};
        for (auto it = lru.begin(); it != lru.end(); ++it)
            if (it->first == key) {
                lru.splice(lru.begin(), lru, it);
                return lru.front().second;
            }
        fntrs_plans* pl = nullptr;
        check(fntrs_gpu_plans_create(ctx, k, n, uint32_t(pos.size()), 1, pos.data(), &pl, stream));
        lru.emplace_front(std::move(key), pl);
        if (lru.size() > kCapacity) {
            sync();  // the evicted plan may still be read by queued work
            fntrs_gpu_plans_destroy(lru.back().second);
            lru.pop_back();
        }
        return pl;
    }
};

Shared& shared();

inline uint32_t next_pow2(uint32_t n) {
    uint32_t m = 1;
    while (m < n) m <<= 1;
    return m;
}

// Fe values -> uint16 words + ascending escape indices (shardio.cpp:131-137).
inline void split(const Fe* v, size_t count, std::vector<uint16_t>& words, std::vector<uint64_t>& esc) {
    words.resize(count);
    esc.clear();
    for (size_t i = 0; i < count; ++i) {
        if (v[i] > 65536) throw SizeMismatch("value " + std::to_string(v[i]) + " outside the field");
        words[i] = v[i] == 65536 ? 0 : uint16_t(v[i]);
        if (v[i] == 65536) esc.push_back(i);
    }
}

// Runs fn(d_in_words, d_in_esc, d_out_words, d_out_esc, d_count) with the
// host arrays staged on the device, then joins the result back into Fe.
template <typename Fn>
std::vector<Fe> run(Shared& S, const std::vector<uint16_t>& in_words, const std::vector<uint64_t>& in_esc,
                    size_t out_count, Fn&& fn) {
    const size_t cap = out_count;  // at most one escape per output symbol
    const size_t b_in = (in_words.size() * 2 + 255) / 256 * 256;
    const size_t b_ie = (in_esc.size() * 8 + 255) / 256 * 256 + 256;
    const size_t b_out = (out_count * 2 + 255) / 256 * 256;
    const size_t b_oe = (cap * 8 + 255) / 256 * 256 + 256;
    char* base = static_cast<char*>(S.scratch(b_in + b_ie + b_out + b_oe + 256));
    auto* d_in = reinterpret_cast<uint16_t*>(base);
    auto* d_ie = reinterpret_cast<uint64_t*>(base + b_in);
    auto* d_out = reinterpret_cast<uint16_t*>(base + b_in + b_ie);
    auto* d_oe = reinterpret_cast<uint64_t*>(base + b_in + b_ie + b_out);
    auto* d_cnt = reinterpret_cast<uint64_t*>(base + b_in + b_ie + b_out + b_oe);
    cudaMemcpyAsync(d_in, in_words.data(), in_words.size() * 2, cudaMemcpyHostToDevice, S.stream);
    if (!in_esc.empty())
        cudaMemcpyAsync(d_ie, in_esc.data(), in_esc.size() * 8, cudaMemcpyHostToDevice, S.stream);
    fn(d_in, in_esc.empty() ? nullptr : d_ie, uint64_t(in_esc.size()), d_out, d_oe, uint64_t(cap), d_cnt);
    std::vector<uint16_t> words(out_count);
    std::vector<uint64_t> esc(cap);
    uint64_t ne = 0;
    cudaMemcpyAsync(words.data(), d_out, out_count * 2, cudaMemcpyDeviceToHost, S.stream);
    cudaMemcpyAsync(&ne, d_cnt, 8, cudaMemcpyDeviceToHost, S.stream);
    if (cap) cudaMemcpyAsync(esc.data(), d_oe, cap * 8, cudaMemcpyDeviceToHost, S.stream);
    S.sync();
    if (ne > cap) throw TooManyEscapes("escape list overflow");
    std::vector<Fe> out(words.begin(), words.end());
    for (uint64_t e = 0; e < ne; ++e) out[esc[e]] = 65536;
    return out;
}


// Stream-ordered device allocation owned for the length of one call.
struct DevBuf {
    void* p = nullptr;
    cudaStream_t st = nullptr;
    DevBuf(size_t bytes, cudaStream_t s) : st(s) {
        if (bytes && cudaMallocAsync(&p, bytes, s) != cudaSuccess) throw Error("fntrs: device allocation failed");
    }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

template <typename T>
void upload(Shared& S, DevBuf& d, const T* h, size_t n) {
    if (n && cudaMemcpyAsync(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice, S.stream) != cudaSuccess)
        throw Error("fntrs: host-to-device copy failed");
}

template <typename T>
void download(Shared& S, T* h, const DevBuf& d, size_t n, size_t offset = 0) {
    if (n && cudaMemcpyAsync(h, d.as<T>() + offset, n * sizeof(T), cudaMemcpyDeviceToHost, S.stream) != cudaSuccess)
        throw Error("fntrs: device-to-host copy failed");
}

// The subproduct tree of `points` built on the device (dropin_aux.cpp); the
// caller holds S.mu.
poly::SubproductTree tree_on_device(Shared& S, const std::vector<Fe>& points);

}  // namespace dropin
}  // namespace fntrs
