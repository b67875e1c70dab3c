// cli.cpp -- `fntrs`, the reference CLI's file encode / decode commands
// (proj/tools/fntrs_main.cpp:108-238, options :413-444) over the batched GPU
// codec. Same arguments, shard and manifest files byte for byte, same exit
// codes (0 ok, 1 usage, 2 fntrs::Error / other failures).
//
//   fntrs encode <input> [-o DIR] -k K -n N [--systematic|--non-systematic] [--seed S] [--path P] [--jobs J]
//   fntrs decode <manifest|dir> -o OUT [--path P] [--jobs J]
//   fntrs bench [--grid k1,k2,..] [-k K] [-n N] [--reps R]   (CSV, batched GPU timing)
//   fntrs selftest [--seed S]
//
// The reference codes S = ceil(ceil(len/2)/k) one-codeword stripes and shard j
// carries symbol j of every stripe. Here that is ONE batched stripe of k
// packets of L >= S symbols (DESIGN 4.9): the file is symbolised on the
// device, encoded by one fntrs_gpu_encode[_systematic] call, and row j of the
// encoded stripe is shard j's payload; decode gathers the k lowest surviving
// shards into packets and runs one plan + one batched decode. --path and
// --jobs are accepted for compatibility (the GPU path is exact for every
// Path; stripes run in parallel on the device).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "fntrs/codec.hpp"
#include "fntrs/errors.hpp"
#include "fntrs/interp.hpp"
#include "fntrs/shardio.hpp"
#include "fntrs_gpu.h"
#include "shard_detail.h"

namespace fs = std::filesystem;
using namespace fntrs;

namespace {

constexpr uint32_t kWidth = 64;  // packet width: a multiple of every fused kernel's tile width

std::vector<uint8_t> read_file(const fs::path& p) {
    std::ifstream in(p, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open " + p.string());
    return std::vector<uint8_t>((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

void write_file(const fs::path& p, const uint8_t* data, size_t n) {
    std::ofstream out(p, std::ios::binary | std::ios::trunc);
    if (!out) throw std::runtime_error("cannot create " + p.string());
    out.write(reinterpret_cast<const char*>(data), std::streamsize(n));
    if (!out) throw std::runtime_error("cannot write " + p.string());
}

struct Gpu {
    fntrs_ctx* ctx = nullptr;
    cudaStream_t st = nullptr;
    std::vector<void*> bufs;
    Gpu() {
        if (fntrs_gpu_create(0, &ctx)) throw Error("fntrs: no usable CUDA device (the codec has no CPU fallback)");
        if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) throw Error("fntrs: cannot create a stream");
    }
    ~Gpu() {  // the context first: its cached plans release on this stream
        if (st) cudaStreamSynchronize(st);
        if (ctx) fntrs_gpu_destroy(ctx);
        for (void* p : bufs) cudaFree(p);
        if (st) cudaStreamDestroy(st);
    }
    template <typename T>
    T* alloc(size_t n) {
        void* p = nullptr;
        if (cudaMalloc(&p, std::max<size_t>(n * sizeof(T), 16))) throw Error("fntrs: device allocation failed");
        bufs.push_back(p);
        return static_cast<T*>(p);
    }
    void check(int rc) {
        if (rc) throw_status(rc, std::string(fntrs_gpu_status_string(rc)) + ": " + fntrs_gpu_last_error(ctx));
    }
    void copy(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
        if (bytes && cudaMemcpyAsync(dst, src, bytes, kind, st)) throw Error("fntrs: copy failed");
    }
    void sync() {
        if (cudaStreamSynchronize(st)) throw Error("fntrs: CUDA error");
    }
};

uint32_t packet_width(uint32_t stripes) { return std::max(kWidth, (stripes + kWidth - 1) / kWidth * kWidth); }

int cmd_encode(const std::string& input, const std::string& outdir, uint32_t k, uint32_t n, bool systematic,
               uint64_t seed) {
    const auto data = read_file(input);
    (void)codec::CodeParams::make(k, n, systematic);  // SizeMismatch as the reference
    const uint64_t chunk_id = seed;
    const uint64_t words = (data.size() + 1) / 2;
    const uint32_t S = uint32_t((words + k - 1) / k), L = packet_width(S);
    Gpu g;
    uint8_t* d_data = g.alloc<uint8_t>(data.size());
    uint16_t* d_src = g.alloc<uint16_t>(size_t(k) * L);
    uint16_t* d_enc = g.alloc<uint16_t>(size_t(n) * L);
    const uint64_t cap = uint64_t(n) * L / 1024 + 4096;
    uint64_t* d_esc = g.alloc<uint64_t>(cap + 1);
    uint8_t* d_be = g.alloc<uint8_t>(size_t(n) * 2 * S);
    g.copy(d_data, data.data(), data.size(), cudaMemcpyHostToDevice);
    g.check(fntrs_gpu_symbolize(g.ctx, d_data, data.size(), k, L, d_src, g.st));
    auto enc = systematic ? fntrs_gpu_encode_systematic : fntrs_gpu_encode;
    g.check(enc(g.ctx, k, n, 1, L, d_src, nullptr, 0, d_enc, d_esc, cap, d_esc + cap, g.st));
    g.check(fntrs_gpu_words_to_be(g.ctx, d_enc, n, L, S, d_be, 2ull * S, g.st));
    std::vector<uint8_t> be(size_t(n) * 2 * S);
    uint64_t ne = 0;
    g.copy(be.data(), d_be, be.size(), cudaMemcpyDeviceToHost);
    g.copy(&ne, d_esc + cap, 8, cudaMemcpyDeviceToHost);
    g.sync();
    if (ne > cap) throw TooManyEscapes("escape list overflow");
    std::vector<uint64_t> esc(ne);
    g.copy(esc.data(), d_esc, ne * 8, cudaMemcpyDeviceToHost);
    g.sync();
    fs::create_directories(outdir);
    shardio::ShardInfo info{chunk_id, k, n, 0, systematic};
    size_t e = 0;
    for (uint32_t j = 0; j < n; ++j) {
        std::vector<uint64_t> row_esc;  // escapes of row j inside the file's S symbols
        for (; e < esc.size() && esc[e] / L == j; ++e)
            if (esc[e] % L < S) row_esc.push_back(esc[e] % L);
        info.shard_index = j;
        std::vector<uint8_t> out = shardio::detail::shard_header(info, S, row_esc);
        out.insert(out.end(), be.begin() + size_t(j) * 2 * S, be.begin() + size_t(j + 1) * 2 * S);
        write_file(fs::path(outdir) / shardio::shard_filename(chunk_id, j), out.data(), out.size());
    }
    const shardio::ChunkManifest manifest{chunk_id, data.size(), k, n, S, systematic};
    const auto mb = shardio::write_manifest(manifest);
    const std::string mname = shardio::manifest_filename(chunk_id);
    write_file(fs::path(outdir) / mname, mb.data(), mb.size());
    std::printf("encode: %llu bytes, k=%u n=%u stripes=%u %s\n", static_cast<unsigned long long>(data.size()), k, n, S,
                systematic ? "systematic" : "non-systematic");
    std::printf("encode: wrote %u shards and %s to %s\n", n, mname.c_str(), outdir.c_str());
    return 0;
}

fs::path resolve_manifest(const fs::path& p) {  // fntrs_main.cpp:165-181
    if (!fs::is_directory(p)) return p;
    fs::path found;
    int count = 0;
    for (const auto& entry : fs::directory_iterator(p))
        if (entry.is_regular_file() && entry.path().filename().string().ends_with(".manifest.fnt")) {
            found = entry.path();
            ++count;
        }
    if (count == 0) throw std::runtime_error("no *.manifest.fnt in " + p.string());
    if (count > 1) throw std::runtime_error("multiple manifests in " + p.string() + "; pass one explicitly");
    return found;
}

int cmd_decode(const std::string& input, const std::string& output) {
    const fs::path mpath = resolve_manifest(input);
    const auto manifest = shardio::read_manifest(read_file(mpath));
    const fs::path dir = mpath.has_parent_path() ? mpath.parent_path() : fs::path(".");
    const uint32_t k = manifest.k, n = manifest.n, S = manifest.stripes, L = packet_width(S);
    (void)codec::CodeParams::make(k, n, manifest.systematic);
    // survivors in ascending position; the decoder uses the k lowest (codec.cpp:85-94)
    std::vector<uint32_t> pos;
    std::vector<uint8_t> be;  // [k][2S] big-endian payload rows
    std::vector<uint64_t> rx_esc;
    uint32_t found = 0;
    for (uint32_t j = 0; j < n; ++j) {
        const fs::path sp = dir / shardio::shard_filename(manifest.chunk_id, j);
        std::error_code ec;
        if (!fs::exists(sp, ec)) continue;
        try {
            const auto bytes = read_file(sp);
            const auto s = shardio::detail::parse_shard(bytes);
            if (s.info.chunk_id != manifest.chunk_id || s.info.k != k || s.info.n != n ||
                s.info.systematic != manifest.systematic || s.info.shard_index != j || s.symbols != S) {
                std::fprintf(stderr, "warning: %s does not match the manifest, skipping\n", sp.string().c_str());
                continue;
            }
            ++found;
            if (pos.size() < k) {
                for (uint32_t e : s.escapes) rx_esc.push_back(uint64_t(pos.size()) * L + e);
                pos.push_back(j);
                be.insert(be.end(), bytes.begin() + s.payload_offset, bytes.begin() + s.payload_offset + 2ull * S);
            }
        } catch (const Error& e) {
            std::fprintf(stderr, "warning: %s unreadable (%s), skipping\n", sp.string().c_str(), e.what());
        }
    }
    if (found < k)
        throw NotEnoughShards("not enough shards: found " + std::to_string(found) + ", required " + std::to_string(k));
    Gpu g;
    uint8_t* d_be = g.alloc<uint8_t>(be.size());
    uint16_t* d_rx = g.alloc<uint16_t>(size_t(k) * L);
    uint64_t* d_rxe = g.alloc<uint64_t>(rx_esc.size());
    uint16_t* d_dec = g.alloc<uint16_t>(size_t(k) * L);
    const uint64_t cap = uint64_t(k) * L / 1024 + 4096;
    uint64_t* d_esc = g.alloc<uint64_t>(cap + 1);
    uint32_t* d_sp = g.alloc<uint32_t>(1);
    uint8_t* d_out = g.alloc<uint8_t>(manifest.original_length);
    g.copy(d_be, be.data(), be.size(), cudaMemcpyHostToDevice);
    g.copy(d_rxe, rx_esc.data(), rx_esc.size() * 8, cudaMemcpyHostToDevice);
    if (cudaMemsetAsync(d_sp, 0, 4, g.st)) throw Error("fntrs: memset failed");
    g.check(fntrs_gpu_be_to_words(g.ctx, d_be, 2ull * S, k, S, L, d_rx, g.st));
    fntrs_plans* pl = nullptr;
    g.check(fntrs_gpu_plans_create(g.ctx, k, n, k, 1, pos.data(), &pl, g.st));
    auto dec = manifest.systematic ? fntrs_gpu_decode_systematic : fntrs_gpu_decode;
    const int rc = dec(g.ctx, pl, 1, L, d_sp, d_rx, rx_esc.empty() ? nullptr : d_rxe, rx_esc.size(), d_dec, d_esc, cap,
                       d_esc + cap, g.st);
    if (!rc) g.check(fntrs_gpu_desymbolize(g.ctx, d_dec, k, L, manifest.original_length, d_out, g.st));
    std::vector<uint8_t> out(manifest.original_length);
    if (!rc) g.copy(out.data(), d_out, out.size(), cudaMemcpyDeviceToHost);
    g.sync();
    fntrs_gpu_plans_destroy(pl);
    g.check(rc);
    write_file(output, out.data(), out.size());
    std::printf("decode: wrote %llu bytes to %s from %u shards\n", static_cast<unsigned long long>(out.size()),
                output.c_str(), found);
    return 0;
}

// ---- bench: the reference CLI's CSV (variant,k,n,bytes,seconds,MBps,fnt_equivalents;
// fntrs_main.cpp:255-303), measured on the batched GPU path: `seconds` is the device time
// per codeword over a batch of 64 stripes x 256 codewords (CUDA events around `reps`
// stream-ordered calls), bytes = 2k of source per codeword, fnt_equivalents from the
// library's transform tally (fntrs_gpu_transform_counts) per codeword.
uint64_t splitmix(uint64_t& s) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

int cmd_bench(const std::vector<std::pair<uint32_t, uint32_t>>& sizes, int reps, uint64_t seed) {
    std::printf("variant,k,n,bytes,seconds,MBps,fnt_equivalents\n");
    Gpu g;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (const auto& [k, n] : sizes) {
        uint32_t nd = 1;
        while (nd < n) nd <<= 1;
        const uint32_t L = 256, S = 64;
        const uint64_t cw = uint64_t(S) * L;
        std::vector<uint16_t> src(size_t(S) * k * L);
        for (auto& w : src) w = uint16_t(splitmix(seed));
        uint16_t* d_src = g.alloc<uint16_t>(src.size());
        uint16_t* d_enc = g.alloc<uint16_t>(size_t(S) * n * L);
        uint16_t* d_rx = g.alloc<uint16_t>(size_t(S) * k * L);
        uint16_t* d_dec = g.alloc<uint16_t>(size_t(S) * k * L);
        const uint64_t cap = uint64_t(S) * n * L / 1024 + 4096;
        uint64_t* d_esc = g.alloc<uint64_t>(cap + 1);
        uint32_t* d_sp = g.alloc<uint32_t>(S);
        g.copy(d_src, src.data(), src.size() * 2, cudaMemcpyHostToDevice);
        if (cudaMemsetAsync(d_sp, 0, S * 4, g.st)) throw Error("fntrs: memset failed");
        // no-shortcut reception as in the reference's bench: position 0 erased, survivors 1..k
        std::vector<uint32_t> pos(k);
        const uint32_t shift = n > k ? 1u : 0u;
        for (uint32_t i = 0; i < k; ++i) pos[i] = i + shift;
        fntrs_plans* pl = nullptr;
        g.check(fntrs_gpu_plans_create(g.ctx, k, n, k, 1, pos.data(), &pl, g.st));
        auto line = [&](const char* variant, auto&& op) {
            uint64_t before[17], after[17];
            op();  // warm (tables, the context's cached systematic plan)
            g.sync();
            g.check(fntrs_gpu_transform_counts(g.ctx, before));
            cudaEventRecord(e0, g.st);
            for (int r = 0; r < reps; ++r) op();
            cudaEventRecord(e1, g.st);
            g.sync();
            g.check(fntrs_gpu_transform_counts(g.ctx, after));
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            double eq = 0;
            for (int e = 0; e < 17; ++e) eq += double(after[e] - before[e]) * double(1u << e);
            const double per = std::max(double(ms) * 1e-3 / reps / double(cw), 1e-15);
            std::printf("%s,%u,%u,%u,%.9e,%.3f,%.3f\n", variant, k, n, 2 * k, per, 2.0 * k / per / 1e6,
                        eq / nd / double(reps) / double(cw));
        };
        line("encode_nonsystematic", [&] {
            g.check(fntrs_gpu_encode(g.ctx, k, n, S, L, d_src, nullptr, 0, d_enc, d_esc, cap, d_esc + cap, g.st));
        });
        line("encode_systematic", [&] {
            g.check(fntrs_gpu_encode_systematic(g.ctx, k, n, S, L, d_src, nullptr, 0, d_enc, d_esc, cap,
                                                d_esc + cap, g.st));
        });
        // received rows = encoded rows shift..shift+k-1 (their rare escapes do not change the timing)
        g.check(fntrs_gpu_encode(g.ctx, k, n, S, L, d_src, nullptr, 0, d_enc, d_esc, cap, d_esc + cap, g.st));
        for (uint32_t s2 = 0; s2 < S; ++s2)
            g.copy(d_rx + size_t(s2) * k * L, d_enc + (size_t(s2) * n + shift) * L, size_t(k) * L * 2,
                   cudaMemcpyDeviceToDevice);
        line("decode_nonsystematic", [&] {
            g.check(fntrs_gpu_decode(g.ctx, pl, S, L, d_sp, d_rx, nullptr, 0, d_dec, d_esc, cap, d_esc + cap, g.st));
        });
        line("decode_systematic", [&] {
            g.check(fntrs_gpu_decode_systematic(g.ctx, pl, S, L, d_sp, d_rx, nullptr, 0, d_dec, d_esc, cap,
                                                d_esc + cap, g.st));
        });
        g.sync();
        fntrs_gpu_plans_destroy(pl);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return 0;
}

// ---- selftest: MDS-exhaustive decoding of small codes, then randomized
// equivalence of the fast interpolation with the quadratic oracle and of every
// encoder / decoder variant (the reference CLI's two suites,
// fntrs_main.cpp:305-405), through the drop-in API on the GPU.
std::vector<Fe> random_fe(uint32_t count, uint64_t& st) {
    std::vector<Fe> v(count);
    for (auto& x : v) x = Fe(splitmix(st) % 65537);
    return v;
}

std::vector<uint32_t> random_subset(uint32_t k, uint32_t n, uint64_t& st) {
    std::vector<uint32_t> all(n);
    for (uint32_t i = 0; i < n; ++i) all[i] = i;
    for (uint32_t i = 0; i < k; ++i) std::swap(all[i], all[i + uint32_t(splitmix(st) % (n - i))]);
    all.resize(k);
    return all;
}

int cmd_selftest(uint64_t seed) {
    uint64_t st = seed;
    bool ok = true;
    const std::pair<uint32_t, uint32_t> codes[] = {{4, 2}, {8, 4}, {8, 5}, {16, 12}};  // (n, k)
    for (const auto& [n, k] : codes) {
        const auto sys = codec::CodeParams::make(k, n, true), non = codec::CodeParams::make(k, n, false);
        const auto src = random_fe(k, st);
        const auto es = codec::encode_systematic(sys, src), en = codec::encode_nonsystematic(non, src);
        uint64_t patterns = 0, failures = 0;
        for (uint32_t mask = 0; mask < (1u << n); ++mask) {
            if (uint32_t(__builtin_popcount(mask)) < k) continue;
            ++patterns;
            codec::Codeword rs, rn;
            for (uint32_t j = 0; j < n; ++j)
                if (mask >> j & 1u) {
                    rs.push_back({j, es[j]});
                    rn.push_back({j, en[j]});
                }
            failures += codec::decode_systematic(sys, rs, codec::Path::Fast) != src ||
                        codec::decode_direct(sys, rs) != src ||
                        codec::decode_nonsystematic(non, rn, codec::Path::Fast) != src ||
                        codec::decode_direct(non, rn) != src;
        }
        std::printf("selftest: mds (%u,%u): %llu patterns, %llu failures\n", n, k,
                    static_cast<unsigned long long>(patterns), static_cast<unsigned long long>(failures));
        ok = ok && failures == 0;
    }
    const int instances = 100;
    int passed = 0;
    for (int t = 0; t < instances; ++t) {
        const uint32_t k = 1 + uint32_t(splitmix(st) % 128);
        uint32_t nd = 2;
        while (nd < k) nd <<= 1;
        if ((splitmix(st) & 1) && nd < 1024) nd <<= 1;
        const auto positions = random_subset(k, nd, st);
        const auto values = random_fe(k, st);
        auto fast = interp::interpolate(interp::build_plan(nd, positions), values);
        std::vector<std::pair<Fe, Fe>> points(k);
        const Fe r = gf::root_of_unity(nd, false);
        for (uint32_t j = 0; j < k; ++j) points[j] = {gf::pow(r, positions[j]), values[j]};
        auto slow = interp::lagrange_oracle(points);
        fast.resize(k, 0);
        slow.resize(k, 0);
        bool good = fast == slow;
        const uint32_t n = k + uint32_t(splitmix(st) % (512 - k + 1));
        const auto sys = codec::CodeParams::make(k, n, true), non = codec::CodeParams::make(k, n, false);
        const auto src = random_fe(k, st);
        const auto es = codec::encode_systematic(sys, src, codec::Path::Fast);
        good = good && es == codec::encode_systematic_direct(sys, src) &&
               es == codec::encode_systematic_intermediate_direct(sys, src);
        const auto en = codec::encode_nonsystematic(non, src);
        const auto keep = random_subset(k, n, st);
        codec::Codeword rs(k), rn(k);
        for (uint32_t j = 0; j < k; ++j) {
            rs[j] = {keep[j], es[keep[j]]};
            rn[j] = {keep[j], en[keep[j]]};
        }
        good = good && codec::decode_systematic(sys, rs, codec::Path::Fast) == src &&
               codec::decode_direct(sys, rs) == src &&
               codec::decode_nonsystematic(non, rn, codec::Path::Fast) == src && codec::decode_direct(non, rn) == src;
        passed += good;
    }
    std::printf("selftest: oracle equivalence: %d/%d instances ok\n", passed, instances);
    ok = ok && passed == instances;
    std::printf("selftest: %s\n", ok ? "PASS" : "FAIL");
    return ok ? 0 : 2;
}

[[noreturn]] void usage(const char* msg) {
    std::fprintf(stderr,
                 "%s\nusage: fntrs encode <input> [-o DIR] -k K -n N [--systematic|--non-systematic] [--seed S]\n"
                 "       fntrs decode <manifest|dir> -o OUT\n"
                 "       fntrs bench [--grid k1,k2,..] [-k K] [-n N] [--reps R] [--seed S]\n"
                 "       fntrs selftest [--seed S]\n",
                 msg);
    std::exit(1);
}

uint64_t to_u64(const std::string& v, const char* what) {
    try {
        size_t used = 0;
        const unsigned long long x = std::stoull(v, &used, 0);
        if (used != v.size()) throw std::invalid_argument(v);
        return x;
    } catch (const std::exception&) {
        usage((std::string("bad value for ") + what + ": " + v).c_str());
    }
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) usage("missing subcommand");
    const std::string cmd = argv[1];
    std::string input, output = ".";
    uint64_t k = 0, n = 0, seed = 1, reps = 5;
    std::vector<uint32_t> grid;
    bool systematic = true, have_out = false, have_k = false, have_n = false;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        auto value = [&](const char* what) -> std::string {
            if (i + 1 >= argc) usage((std::string("missing value for ") + what).c_str());
            return argv[++i];
        };
        if (a == "-o" || a == "--out") output = value("--out"), have_out = true;
        else if (a == "-k" || a == "--k") k = to_u64(value("--k"), "--k"), have_k = true;
        else if (a == "-n" || a == "--n") n = to_u64(value("--n"), "--n"), have_n = true;
        else if (a == "--seed") seed = to_u64(value("--seed"), "--seed");
        else if (a == "--systematic") systematic = true;
        else if (a == "--non-systematic") systematic = false;
        else if (a == "--path") {
            const std::string p = value("--path");
            if (p != "auto" && p != "fast" && p != "direct") usage("--path must be auto, fast or direct");
        } else if (a == "--jobs") (void)to_u64(value("--jobs"), "--jobs");
        else if (a == "--reps") reps = to_u64(value("--reps"), "--reps");
        else if (a == "--grid") {
            const std::string gs = value("--grid");
            for (size_t p = 0; p <= gs.size();) {
                const size_t q = std::min(gs.find(',', p), gs.size());
                grid.push_back(uint32_t(to_u64(gs.substr(p, q - p), "--grid")));
                p = q + 1;
            }
        }
        else if (!a.empty() && a[0] == '-') usage(("unknown option " + a).c_str());
        else if (input.empty()) input = a;
        else usage(("unexpected argument " + a).c_str());
    }
    try {
        if (cmd == "encode") {
            if (input.empty() || !have_k || !have_n) usage("encode needs <input>, --k and --n");
            if (k < 1 || k > n || n > 65536) usage("need 1 <= k <= n <= 65536");
            if (k == 65536) usage("k = 65536 does not fit the shard header");
            return cmd_encode(input, output, uint32_t(k), uint32_t(n), systematic, seed);
        }
        if (cmd == "decode") {
            if (input.empty() || !have_out) usage("decode needs <input> and --out");
            return cmd_decode(input, output);
        }
        if (cmd == "bench") {  // fntrs_main.cpp:444-472: a grid of k (n = 2k), one size, or a default set
            std::vector<std::pair<uint32_t, uint32_t>> sizes;
            if (!grid.empty()) {
                for (uint32_t g : grid) {
                    if (g < 1 || g > 32768) usage("grid k values must be in [1, 32768]");
                    sizes.emplace_back(g, 2 * g);
                }
            } else if (!have_k && !have_n) {
                sizes = {{256, 512}, {1024, 2048}, {4096, 8192}};
            } else {
                if (!have_n) n = 2 * k;
                if (!have_k) k = n / 2;
                if (k < 1 || k > n || n > 65536) usage("need 1 <= k <= n <= 65536");
                sizes = {{uint32_t(k), uint32_t(n)}};
            }
            if (reps < 1) usage("--reps must be positive");
            return cmd_bench(sizes, int(reps), seed);
        }
        if (cmd == "selftest") return cmd_selftest(seed);
        usage(("unknown subcommand " + cmd).c_str());
    } catch (const Error& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
}
