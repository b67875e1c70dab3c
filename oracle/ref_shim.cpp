// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference library, compiled
// from /root/reference/proj/src with -Dfntrs=fntrs_ref (oracle/Makefile) into
// oracle/_ref/libfntrs_ref.so. Used by tests/ to pin the oracle restatement
// against the reference itself, and by bench.py (--impl reference and the
// cpu_baseline leg) to time the reference's own CPU codec on the host.
//
// The batched entry points mirror the reference CLI's codeword loop:
// gather column j of packet-major stripes, call codec::encode_nonsystematic /
// decode_nonsystematic once per codeword, scatter the result
// (proj/tools/fntrs_main.cpp:122-139,222-231), on `threads` workers pulling
// codeword indices from an atomic counter like for_each_stripe (:72-106).
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

#include "fntrs/codec.hpp"
#include "fntrs/errors.hpp"
#include "fntrs/interp.hpp"
#include "fntrs/shardio.hpp"
#include "fntrs/transform.hpp"

using namespace fntrs;

namespace {

int status_of(const std::exception& e) {
    if (dynamic_cast<const ZeroInverse*>(&e)) return 2;
    if (dynamic_cast<const InvalidTransformSize*>(&e)) return 3;
    if (dynamic_cast<const SizeMismatch*>(&e)) return 4;
    if (dynamic_cast<const ProductTooLarge*>(&e)) return 5;
    if (dynamic_cast<const DuplicatePoint*>(&e)) return 6;
    if (dynamic_cast<const DuplicatePosition*>(&e)) return 7;
    if (dynamic_cast<const PositionOutOfRange*>(&e)) return 8;
    if (dynamic_cast<const TooFewPositions*>(&e)) return 9;
    if (dynamic_cast<const NotEnoughSymbols*>(&e)) return 10;
    if (dynamic_cast<const TooManyEscapes*>(&e)) return 11;
    if (dynamic_cast<const BadMagic*>(&e)) return 12;
    if (dynamic_cast<const BadVersion*>(&e)) return 13;
    if (dynamic_cast<const TruncatedShard*>(&e)) return 14;
    if (dynamic_cast<const MalformedEscapes*>(&e)) return 15;
    if (dynamic_cast<const MalformedHeader*>(&e)) return 16;
    if (dynamic_cast<const LengthMismatch*>(&e)) return 17;
    if (dynamic_cast<const NotEnoughShards*>(&e)) return 18;
    return 1;
}

codec::Path path_of(int p) {
    return p == 1 ? codec::Path::Fast : p == 2 ? codec::Path::Direct : codec::Path::Auto;
}

uint32_t fetch(const uint16_t* base, const uint64_t* esc, uint64_t ne, uint64_t row, uint32_t col,
               uint32_t L) {
    uint16_t w = base[row * L + col];
    if (w || !ne) return w;
    const uint64_t key = row * L + col;
    return std::binary_search(esc, esc + ne, key) ? 65536u : 0u;
}

template <typename Fn>
int run_parallel(uint64_t items, unsigned threads, Fn&& fn) {
    threads = std::max(1u, threads);
    std::atomic<uint64_t> next{0};
    std::atomic<int> status{0};
    auto worker = [&](unsigned w) {
        for (;;) {
            uint64_t t = next.fetch_add(1);
            if (t >= items || status.load()) return;
            try {
                fn(w, t);
            } catch (const std::exception& e) {
                int expected = 0;
                status.compare_exchange_strong(expected, status_of(e));
                return;
            }
        }
    };
    if (threads == 1) {
        worker(0);
    } else {
        std::vector<std::thread> pool;
        for (unsigned w = 0; w < threads; ++w) pool.emplace_back(worker, w);
        for (auto& th : pool) th.join();
    }
    return status.load();
}

}  // namespace

extern "C" {

int ref_fnt_forward(uint32_t n, const uint32_t* in, uint32_t* out) {
    try {
        auto v = fnt_forward(plan_for(n), std::span<const Fe>(in, n));
        std::copy(v.begin(), v.end(), out);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_fnt_inverse(uint32_t n, const uint32_t* in, uint32_t* out) {
    try {
        auto v = fnt_inverse(plan_for(n), std::span<const Fe>(in, n));
        std::copy(v.begin(), v.end(), out);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_encode(uint32_t k, uint32_t n, uint32_t src_len, const uint32_t* src, uint32_t* out) {
    try {
        auto params = codec::CodeParams::make(k, n, false);
        auto v = codec::encode_nonsystematic(params, std::span<const Fe>(src, src_len));
        std::copy(v.begin(), v.end(), out);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_decode(uint32_t k, uint32_t n, uint32_t count, const uint32_t* pos, const uint32_t* val,
               int path, uint32_t* out) {
    try {
        auto params = codec::CodeParams::make(k, n, false);
        codec::Codeword rx(count);
        for (uint32_t i = 0; i < count; ++i) rx[i] = {pos[i], val[i]};
        auto v = codec::decode_nonsystematic(params, rx, path_of(path));
        std::copy(v.begin(), v.end(), out);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// Systematic codec (proj/src/codec.cpp:151-196), reference-default path selection.
int ref_encode_systematic(uint32_t k, uint32_t n, uint32_t src_len, const uint32_t* src, int path,
                          uint32_t* out) {
    try {
        auto params = codec::CodeParams::make(k, n, true);
        auto v = codec::encode_systematic(params, std::span<const Fe>(src, src_len), path_of(path));
        std::copy(v.begin(), v.end(), out);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_decode_systematic(uint32_t k, uint32_t n, uint32_t count, const uint32_t* pos, const uint32_t* val,
                          int path, uint32_t* out) {
    try {
        auto params = codec::CodeParams::make(k, n, true);
        codec::Codeword rx(count);
        for (uint32_t i = 0; i < count; ++i) rx[i] = {pos[i], val[i]};
        auto v = codec::decode_systematic(params, rx, path_of(path));
        std::copy(v.begin(), v.end(), out);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// DecodePlan fields (proj/include/fntrs/interp.hpp:18-32).
int ref_build_plan(uint32_t n, uint32_t k, const uint32_t* positions, uint32_t* a_out,
                   uint32_t* a_len, uint32_t* aprime_inv, uint32_t* product_size,
                   uint32_t* a_fnt) {
    try {
        auto plan = interp::build_plan(n, std::span<const uint32_t>(positions, k));
        const auto& a = plan.a();
        *a_len = static_cast<uint32_t>(a.size());
        std::copy(a.begin(), a.end(), a_out);
        std::copy(plan.aprime_at_x_inv.begin(), plan.aprime_at_x_inv.end(), aprime_inv);
        *product_size = plan.product_size;
        if (a_fnt) std::copy(plan.a_fnt.begin(), plan.a_fnt.end(), a_fnt);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// Which codec the batched stripe loops run: 0 non-systematic (default), 1 the
// systematic pair (encode_systematic / decode_systematic, the CLI default mode,
// proj/tools/fntrs_main.cpp:413).
static std::atomic<int> g_systematic{0};
void ref_set_systematic(int on) { g_systematic = on; }

// CLI-style batched encode over packet-major stripes. Returns the escape
// count (sorted symbol indices row*L+col in out_esc) or a negative status.
int64_t ref_encode_stripes(uint32_t k, uint32_t n, uint32_t stripes, uint32_t L,
                           const uint16_t* src, const uint64_t* src_esc, uint64_t n_src_esc,
                           uint16_t* out, uint64_t* out_esc, uint64_t esc_cap, unsigned threads) {
    codec::CodeParams params;
    try {
        params = codec::CodeParams::make(k, n, false);
    } catch (const std::exception& e) {
        return -status_of(e);
    }
    std::mutex mu;
    std::vector<uint64_t> escapes;
    const bool sys = g_systematic.load() != 0;
    int st = run_parallel(uint64_t(stripes) * L, threads, [&](unsigned, uint64_t t) {
        const uint32_t s = uint32_t(t / L), j = uint32_t(t % L);
        std::vector<Fe> col(k);
        for (uint32_t i = 0; i < k; ++i) col[i] = fetch(src, src_esc, n_src_esc, uint64_t(s) * k + i, j, L);
        std::vector<Fe> enc = sys ? codec::encode_systematic(params, col) : codec::encode_nonsystematic(params, col);
        for (uint32_t i = 0; i < n; ++i) {
            const uint64_t row = uint64_t(s) * n + i;
            out[row * L + j] = enc[i] == 65536 ? 0 : uint16_t(enc[i]);
            if (enc[i] == 65536) {
                std::lock_guard<std::mutex> lock(mu);
                escapes.push_back(row * L + j);
            }
        }
    });
    if (st) return -st;
    if (escapes.size() > esc_cap) return -11;
    std::sort(escapes.begin(), escapes.end());
    std::copy(escapes.begin(), escapes.end(), out_esc);
    return int64_t(escapes.size());
}

// CLI-style batched decode; each stripe s uses pattern stripe_pattern[s]
// (k ascending positions), rx rows s*k+i carry the packet at position i of
// that pattern. path: 0 Auto, 1 Fast, 2 Direct (codec.hpp:39).
int64_t ref_decode_stripes(uint32_t k, uint32_t n, uint32_t stripes, uint32_t L,
                           uint32_t npatterns, const uint32_t* patterns,
                           const uint32_t* stripe_pattern, const uint16_t* rx,
                           const uint64_t* rx_esc, uint64_t n_rx_esc, uint16_t* out,
                           uint64_t* out_esc, uint64_t esc_cap, int path, unsigned threads) {
    codec::CodeParams params;
    try {
        params = codec::CodeParams::make(k, n, false);
    } catch (const std::exception& e) {
        return -status_of(e);
    }
    for (uint32_t s = 0; s < stripes; ++s)
        if (stripe_pattern[s] >= npatterns) return -1;
    std::mutex mu;
    std::vector<uint64_t> escapes;
    const codec::Path p = path_of(path);
    const bool sys = g_systematic.load() != 0;
    int st = run_parallel(uint64_t(stripes) * L, threads, [&](unsigned, uint64_t t) {
        const uint32_t s = uint32_t(t / L), j = uint32_t(t % L);
        const uint32_t* pos = patterns + uint64_t(stripe_pattern[s]) * k;
        codec::Codeword cw(k);
        for (uint32_t i = 0; i < k; ++i)
            cw[i] = {pos[i], fetch(rx, rx_esc, n_rx_esc, uint64_t(s) * k + i, j, L)};
        std::vector<Fe> dec = sys ? codec::decode_systematic(params, cw, p) : codec::decode_nonsystematic(params, cw, p);
        for (uint32_t i = 0; i < k; ++i) {
            const uint64_t row = uint64_t(s) * k + i;
            out[row * L + j] = dec[i] == 65536 ? 0 : uint16_t(dec[i]);
            if (dec[i] == 65536) {
                std::lock_guard<std::mutex> lock(mu);
                escapes.push_back(row * L + j);
            }
        }
    });
    if (st) return -st;
    if (escapes.size() > esc_cap) return -11;
    std::sort(escapes.begin(), escapes.end());
    std::copy(escapes.begin(), escapes.end(), out_esc);
    return int64_t(escapes.size());
}

// The reference CLI's encode (proj/tools/fntrs_main.cpp:117-160) minus the
// file system: symbolize, per-stripe encode, one shard per code position,
// manifest. Writes the manifest then shards 0..n-1 back to back into out
// (capacity cap) and their sizes into sizes[0..n]; returns total bytes or a
// negative status.
int64_t ref_encode_file(const uint8_t* data, uint64_t len, uint32_t k, uint32_t n, int systematic,
                        uint64_t chunk_id, uint8_t* out, uint64_t cap, uint64_t* sizes) {
    try {
        const auto params = codec::CodeParams::make(k, n, systematic != 0);
        const auto m = shardio::symbolize(std::span<const uint8_t>(data, len), k);
        std::vector<Fe> enc(size_t(m.stripes) * n);
        for (uint32_t t = 0; t < m.stripes; ++t) {
            std::span<const Fe> src(m.cells.data() + size_t(t) * k, k);
            auto row = systematic ? codec::encode_systematic(params, src) : codec::encode_nonsystematic(params, src);
            std::copy(row.begin(), row.end(), enc.begin() + size_t(t) * n);
        }
        uint64_t pos = 0;
        auto emit = [&](const std::vector<uint8_t>& b, uint64_t* sz) {
            if (pos + b.size() > cap) throw TooManyEscapes("output capacity");
            std::memcpy(out + pos, b.data(), b.size());
            pos += b.size();
            *sz = b.size();
        };
        emit(shardio::write_manifest({chunk_id, len, k, n, m.stripes, systematic != 0}), &sizes[0]);
        shardio::ShardInfo info{chunk_id, k, n, 0, systematic != 0};
        std::vector<Fe> payload(m.stripes);
        for (uint32_t j = 0; j < n; ++j) {
            for (uint32_t t = 0; t < m.stripes; ++t) payload[t] = enc[size_t(t) * n + j];
            info.shard_index = j;
            emit(shardio::write_shard(info, payload), &sizes[1 + j]);
        }
        return int64_t(pos);
    } catch (const std::exception& e) {
        return -status_of(e);
    }
}

// shardio::write_shard of explicit values (frozen-layout checks)
int64_t ref_write_shard(uint64_t chunk_id, uint32_t k, uint32_t n, uint32_t index, int systematic,
                        const uint32_t* payload, uint64_t count, uint8_t* out, uint64_t cap) {
    try {
        auto b = shardio::write_shard({chunk_id, k, n, index, systematic != 0},
                                      std::span<const Fe>(payload, count));
        if (b.size() > cap) return -1;
        std::memcpy(out, b.data(), b.size());
        return int64_t(b.size());
    } catch (const std::exception& e) {
        return -status_of(e);
    }
}

// shardio::read_shard status (0 = accepted) for malformed-input checks
int ref_read_shard_status(const uint8_t* bytes, uint64_t len) {
    try {
        (void)shardio::read_shard(std::span<const uint8_t>(bytes, len));
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_has_avx2(void) {
#if defined(__x86_64__)
    return __builtin_cpu_supports("avx2") ? 1 : 0;
#else
    return 0;
#endif
}

}  // extern "C"
