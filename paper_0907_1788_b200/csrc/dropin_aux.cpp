// dropin_aux.cpp -- the reference's poly layer (include/fntrs/poly.hpp) and
// shard wire format (include/fntrs/shardio.hpp) for the drop-in API.
//
// Polynomial arithmetic runs on the device (csrc/poly_aux.cu through the C
// ABI); the shard format's header fields and checks are host byte formatting
// in the order of the reference (proj/src/shardio.cpp:83-273), with payload
// words converted to / from big-endian bytes by the device kernels of
// csrc/shards.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <map>
#include <string>
#include <vector>

#include "dropin_shared.h"
#include "fntrs/errors.hpp"
#include "fntrs/geom.hpp"
#include "fntrs/poly.hpp"
#include "fntrs/shardio.hpp"
#include "fntrs_gpu.h"
#include "shard_detail.h"

namespace fntrs {
namespace dropin {

poly::SubproductTree tree_on_device(Shared& S, const std::vector<Fe>& points) {
    const uint32_t k = uint32_t(points.size());
    uint32_t levels = 0;
    uint64_t nodes = 0, coeffs = 0;
    S.check(fntrs_gpu_subproduct_tree_layout(k, &levels, nullptr, 0, nullptr, &nodes, &coeffs));
    std::vector<uint32_t> level_nodes(levels), node_len(nodes);
    S.check(fntrs_gpu_subproduct_tree_layout(k, &levels, level_nodes.data(), levels, node_len.data(), &nodes, &coeffs));
    DevBuf d((k + coeffs) * 4, S.stream);
    upload(S, d, points.data(), k);
    S.check(fntrs_gpu_subproduct_tree(S.ctx, k, d.as<uint32_t>(), d.as<uint32_t>() + k, S.stream));
    std::vector<Fe> all(coeffs);
    download(S, all.data(), d, coeffs, k);
    S.sync();
    poly::SubproductTree t;
    size_t node = 0, off = 0;
    for (uint32_t l = 0; l < levels; ++l) {
        std::vector<poly::Poly> lv(level_nodes[l]);
        for (auto& p : lv) {
            p.assign(all.begin() + off, all.begin() + off + node_len[node]);
            off += node_len[node++];
        }
        t.levels.push_back(std::move(lv));
    }
    return t;
}

}  // namespace dropin

using namespace dropin;

// ---- poly.hpp ---------------------------------------------------------------
namespace poly {

void normalize(Poly& p) {
    while (!p.empty() && p.back() == 0) p.pop_back();
}

namespace {
// raw product on the device (length la + lb - 1), normalised
Poly product(std::span<const Fe> a, std::span<const Fe> b) {
    if (a.empty() || b.empty()) return {};
    const size_t la = a.size(), lb = b.size(), lo = la + lb - 1;
    Shared& S = shared();
    std::lock_guard<std::mutex> lock(S.mu);
    S.ensure();
    DevBuf d((la + lb + lo) * 4, S.stream);
    upload(S, d, a.data(), la);
    if (cudaMemcpyAsync(d.as<uint32_t>() + la, b.data(), lb * 4, cudaMemcpyHostToDevice, S.stream) != cudaSuccess)
        throw Error("fntrs: host-to-device copy failed");
    const fntrs_poly_pair pr{0, la, la + lb, uint32_t(la), uint32_t(lb)};
    S.check(fntrs_gpu_poly_products(S.ctx, 1, &pr, d.as<uint32_t>(), d.as<uint32_t>(), S.stream));
    Poly out(lo);
    download(S, out.data(), d, lo, la + lb);
    S.sync();
    normalize(out);
    return out;
}

void check_transform_bound(size_t la, size_t lb) {  // poly.cpp: the transform tier's limit
    if (la && lb && la + lb - 1 > 65536)
        throw ProductTooLarge("product needs " + std::to_string(la + lb - 1) +
                              " coefficients, the largest transform is 65536");
}
}  // namespace

Poly mul_schoolbook(std::span<const Fe> a, std::span<const Fe> b) { return product(a, b); }
Poly mul_karatsuba(std::span<const Fe> a, std::span<const Fe> b) { return product(a, b); }

Poly mul_fnt(std::span<const Fe> a, std::span<const Fe> b) {
    check_transform_bound(a.size(), b.size());
    return product(a, b);
}

Poly mul(std::span<const Fe> a, std::span<const Fe> b, const MulTuning& tuning) {
    const size_t lo = (a.empty() || b.empty()) ? 0 : a.size() + b.size() - 1;
    if (lo >= tuning.karatsuba_below) check_transform_bound(a.size(), b.size());  // the transform tier
    return product(a, b);
}

Poly mul_low(std::span<const Fe> a, std::span<const Fe> b, std::size_t count, const MulTuning&) {
    std::span<const Fe> at = a.first(std::min(count, a.size()));
    std::span<const Fe> bt = b.first(std::min(count, b.size()));
    Poly out = product(at, bt);  // exact at any length on the device: no split needed
    if (out.size() > count) out.resize(count);
    normalize(out);
    return out;
}

std::vector<Fe> middle_product(std::span<const Fe> a, std::span<const Fe> b) {  // poly.cpp:171-199
    const size_t n = a.size();
    if (n == 0 || (n & (n - 1)) != 0)
        throw SizeMismatch("middle product needs a power-of-two short operand, got " + std::to_string(n));
    if (b.size() != 2 * n - 1)
        throw SizeMismatch("middle product long operand must have " + std::to_string(2 * n - 1) + " entries, got " +
                           std::to_string(b.size()));
    if (2 * n > 65536)
        throw ProductTooLarge("middle product needs a size-" + std::to_string(2 * n) + " transform, limit is 65536");
    Poly full = product(a, b);
    full.resize(3 * n - 2, 0);
    return std::vector<Fe>(full.begin() + (n - 1), full.begin() + (2 * n - 1));
}

Poly derivative(std::span<const Fe> a) {
    if (a.size() <= 1) return {};
    Shared& S = shared();
    std::lock_guard<std::mutex> lock(S.mu);
    S.ensure();
    DevBuf d((2 * a.size()) * 4, S.stream);
    upload(S, d, a.data(), a.size());
    S.check(fntrs_gpu_poly_derivative(S.ctx, uint32_t(a.size()), d.as<uint32_t>(), d.as<uint32_t>() + a.size(),
                                      S.stream));
    Poly out(a.size() - 1);
    download(S, out.data(), d, out.size(), a.size());
    S.sync();
    normalize(out);
    return out;
}

Fe eval_horner(std::span<const Fe> a, Fe x) {
    Shared& S = shared();
    std::lock_guard<std::mutex> lock(S.mu);
    S.ensure();
    DevBuf d((a.size() + 1) * 4, S.stream);
    upload(S, d, a.data(), a.size());
    S.check(fntrs_gpu_poly_eval(S.ctx, uint32_t(a.size()), d.as<uint32_t>(), x, d.as<uint32_t>() + a.size(),
                                S.stream));
    Fe v = 0;
    download(S, &v, d, 1, a.size());
    S.sync();
    return v;
}

SubproductTree build_subproduct_tree(std::span<const Fe> points) {  // poly.cpp:216-242 checks
    if (points.empty()) throw Error("subproduct tree needs at least one point");
    {
        std::vector<Fe> sorted(points.begin(), points.end());
        std::sort(sorted.begin(), sorted.end());
        auto dup = std::adjacent_find(sorted.begin(), sorted.end());
        if (dup != sorted.end()) throw DuplicatePoint("point " + std::to_string(*dup) + " repeats");
    }
    Shared& S = shared();
    std::lock_guard<std::mutex> lock(S.mu);
    S.ensure();
    return tree_on_device(S, std::vector<Fe>(points.begin(), points.end()));
}

}  // namespace poly

// ---- geom.hpp ---------------------------------------------------------------
namespace geom {

ChirpTable build_chirp(std::uint32_t n, Fe root) {  // geom.cpp:13-41
    ChirpTable t;
    t.n = n;
    t.root = root;
    Shared& S = shared();
    std::lock_guard<std::mutex> lock(S.mu);
    S.ensure();
    if (n == 65536) {
        S.check(fntrs_gpu_chirp_table(S.ctx, n, root, nullptr, nullptr, nullptr, S.stream));  // validates only
        t.full_domain = true;
        return t;
    }
    if (n == 0 || n > 65536 || (n & (n - 1))) S.check(fntrs_gpu_chirp_table(S.ctx, n, root, nullptr, nullptr, nullptr,
                                                                          S.stream));  // throws
    DevBuf d(size_t(5) * n * 4, S.stream);
    uint32_t* p = d.as<uint32_t>();
    S.check(fntrs_gpu_chirp_table(S.ctx, n, root, p, p + 2 * n, p + 3 * n, S.stream));
    t.b.resize(2 * n - 1);
    t.b_inverse.resize(n);
    std::vector<Fe> spec(2 * n);
    download(S, t.b.data(), d, 2 * n - 1, 0);
    download(S, t.b_inverse.data(), d, n, 2 * n);
    download(S, spec.data(), d, 2 * n, 3 * n);
    S.sync();
    S.note_transforms();
    // dif_forward leaves the spectrum in bit-reversed order (transform.hpp)
    t.b_fnt.resize(2 * n);
    uint32_t lg = 0;
    while ((1u << lg) < 2 * n) ++lg;
    for (uint32_t i = 0; i < 2 * n; ++i) {
        uint32_t r = 0;
        for (uint32_t bit = 0; bit < lg; ++bit) r |= ((i >> bit) & 1u) << (lg - 1 - bit);
        t.b_fnt[i] = spec[r];
    }
    return t;
}

std::shared_ptr<const ChirpTable> chirp_for(std::uint32_t n, Fe root) {  // geom.cpp:43-53
    static std::mutex mu;
    static std::map<std::pair<std::uint32_t, Fe>, std::shared_ptr<const ChirpTable>> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({n, root});
    if (it != cache.end()) return it->second;
    auto t = std::make_shared<const ChirpTable>(build_chirp(n, root));
    cache.emplace(std::make_pair(n, root), t);
    return t;
}

namespace {
// a(root^i) on the device with a table's b_inverse and its spectrum (natural
// order: the inverse of dif_forward's bit reversal); full-domain tables have none
std::vector<Fe> eval_with_table(std::span<const Fe> a, const ChirpTable& t, bool negative, Fe root) {
    const uint32_t n = t.n, m = 2 * n;
    Shared& S = shared();
    std::lock_guard<std::mutex> lock(S.mu);
    S.ensure();
    const bool tab = !t.full_domain && t.b_inverse.size() == n && t.b_fnt.size() == m;
    DevBuf d((a.size() + n + (tab ? n + m : 0) + 1) * 4, S.stream);
    uint32_t* p = d.as<uint32_t>();
    upload(S, d, a.data(), a.size());
    uint32_t *binv = nullptr, *spec = nullptr;
    if (tab) {
        binv = p + a.size() + n;
        spec = binv + n;
        std::vector<Fe> nat(m);
        uint32_t lg = 0;
        while ((1u << lg) < m) ++lg;
        for (uint32_t i = 0; i < m; ++i) {
            uint32_t r = 0;
            for (uint32_t bit = 0; bit < lg; ++bit) r |= ((i >> bit) & 1u) << (lg - 1 - bit);
            nat[r] = t.b_fnt[i];
        }
        if (cudaMemcpyAsync(binv, t.b_inverse.data(), size_t(n) * 4, cudaMemcpyHostToDevice, S.stream) ||
            cudaMemcpyAsync(spec, nat.data(), size_t(m) * 4, cudaMemcpyHostToDevice, S.stream))
            throw Error("fntrs: host-to-device copy failed");
        S.sync();  // `nat` is a host temporary
    }
    if (negative)
        S.check(fntrs_gpu_geom_eval_negative(S.ctx, n, root, p, uint32_t(a.size()), binv, spec, p + a.size(),
                                             S.stream));
    else
        S.check(fntrs_gpu_geom_eval(S.ctx, n, t.root, p, uint32_t(a.size()), binv, spec, p + a.size(), S.stream));
    std::vector<Fe> out(n);
    download(S, out.data(), d, n, a.size());
    S.sync();
    S.note_transforms();
    return out;
}
}  // namespace

std::vector<Fe> geom_eval(std::span<const Fe> a, const ChirpTable& table) {  // geom.cpp:75-99
    if (a.size() > table.n) throw SizeMismatch("geom_eval: polynomial has more coefficients than points");
    return eval_with_table(a, table, false, table.root);
}

std::vector<Fe> geom_eval_negative(std::span<const Fe> a, std::uint32_t n, Fe root) {  // geom.cpp:101-116
    if (a.size() > n) throw SizeMismatch("geom_eval_negative: polynomial has more coefficients than points");
    // the table of rho = 1/root, cached like the reference's chirp_for
    return eval_with_table(a, *chirp_for(n, gf::inv(root)), true, root);
}

}  // namespace geom

// ---- shardio.hpp ------------------------------------------------------------
namespace shardio {

namespace {
constexpr uint8_t kShardMagic[4] = {'F', 'N', 'T', 'C'};
constexpr uint8_t kManifestMagic[4] = {'F', 'N', 'T', 'M'};
constexpr uint8_t kVersion = 1;
constexpr uint8_t kSystematicFlag = 0x01;
constexpr size_t kShardHeader = 26, kManifestBytes = 30;

// big-endian field writer / bounds-checked reader
struct BeOut {
    std::vector<uint8_t>& b;
    void u(uint64_t v, int bytes) {
        for (int i = bytes - 1; i >= 0; --i) b.push_back(uint8_t(v >> (8 * i)));
    }
};
struct BeIn {
    std::span<const uint8_t> b;
    size_t at = 0;
    void need(size_t count) const {
        if (at + count > b.size())
            throw TruncatedShard("need " + std::to_string(count) + " more bytes at offset " + std::to_string(at) +
                                 ", have " + std::to_string(b.size() - at));
    }
    uint64_t u(int bytes) {
        need(size_t(bytes));
        uint64_t v = 0;
        for (int i = 0; i < bytes; ++i) v = (v << 8) | b[at + i];
        at += size_t(bytes);
        return v;
    }
    void magic(const uint8_t (&m)[4]) {
        need(4);
        if (!std::equal(m, m + 4, b.begin() + at)) throw BadMagic("unrecognized file magic");
        at += 4;
    }
};

uint16_t n_wire(uint32_t n) { return n == 65536 ? 0 : uint16_t(n); }
uint32_t n_unwire(uint64_t w) { return w == 0 ? 65536u : uint32_t(w); }

// words[i] (host) <-> big-endian bytes through the device kernels
void words_to_be(const std::vector<uint16_t>& words, uint8_t* out) {
    const size_t n = words.size();
    if (!n) return;
    Shared& S = shared();
    std::lock_guard<std::mutex> lock(S.mu);
    S.ensure();
    DevBuf d(n * 2 + n * 2 + 16, S.stream);
    upload(S, d, words.data(), n);
    uint8_t* db = d.as<uint8_t>() + n * 2;
    S.check(fntrs_gpu_words_to_be(S.ctx, d.as<uint16_t>(), 1, uint32_t(n), uint32_t(n), db, n * 2, S.stream));
    if (cudaMemcpyAsync(out, db, n * 2, cudaMemcpyDeviceToHost, S.stream) != cudaSuccess)
        throw Error("fntrs: device-to-host copy failed");
    S.sync();
}

std::vector<uint16_t> be_to_words(const uint8_t* in, size_t n) {
    std::vector<uint16_t> words(n);
    if (!n) return words;
    Shared& S = shared();
    std::lock_guard<std::mutex> lock(S.mu);
    S.ensure();
    DevBuf d(n * 2 + n * 2 + 16, S.stream);
    upload(S, d, in, n * 2);
    uint16_t* dw = reinterpret_cast<uint16_t*>(d.as<uint8_t>() + n * 2);
    S.check(fntrs_gpu_be_to_words(S.ctx, d.as<uint8_t>(), n * 2, 1, uint32_t(n), uint32_t(n), dw, S.stream));
    if (cudaMemcpyAsync(words.data(), dw, n * 2, cudaMemcpyDeviceToHost, S.stream) != cudaSuccess)
        throw Error("fntrs: device-to-host copy failed");
    S.sync();
    return words;
}
}  // namespace

SymbolMatrix symbolize(std::span<const std::uint8_t> data, std::uint32_t k) {
    if (k == 0) throw SizeMismatch("symbolize needs k >= 1");
    SymbolMatrix m;
    m.k = k;
    const uint64_t words = (data.size() + 1) / 2;
    m.stripes = uint32_t((words + k - 1) / k);
    const size_t cells = size_t(m.stripes) * k;
    std::vector<uint8_t> padded(cells * 2, 0);  // the odd last byte and the tail stripe padded with zeros
    std::copy(data.begin(), data.end(), padded.begin());
    const std::vector<uint16_t> w = be_to_words(padded.data(), cells);
    m.cells.assign(w.begin(), w.end());
    return m;
}

std::vector<std::uint8_t> desymbolize(const SymbolMatrix& m, std::uint64_t original_length) {
    const uint64_t capacity = uint64_t(m.stripes) * m.k * 2;
    if (original_length > capacity)
        throw LengthMismatch("length " + std::to_string(original_length) + " exceeds matrix capacity " +
                             std::to_string(capacity));
    const uint64_t words = (original_length + 1) / 2;
    const uint64_t stripes = m.k == 0 ? 0 : (words + m.k - 1) / m.k;
    if (stripes != m.stripes)
        throw LengthMismatch("length " + std::to_string(original_length) + " implies " + std::to_string(stripes) +
                             " stripes, matrix has " + std::to_string(m.stripes));
    std::vector<uint16_t> w(words);
    for (uint64_t i = 0; i < words; ++i) w[i] = uint16_t(m.cells[i]);  // symbols of a matrix are < 65536
    std::vector<uint8_t> out(words * 2);
    words_to_be(w, out.data());
    out.resize(original_length);
    return out;
}

namespace detail {
std::vector<uint8_t> shard_header(const ShardInfo& info, uint64_t symbols, const std::vector<uint64_t>& esc) {
    if (info.k < 1 || info.k > 65535)
        throw SizeMismatch("shard header k must be in [1, 65535], got " + std::to_string(info.k));
    if (info.n < info.k || info.n > 65536)
        throw SizeMismatch("shard header n must be in [k, 65536], got " + std::to_string(info.n));
    if (info.shard_index >= info.n)
        throw SizeMismatch("shard index " + std::to_string(info.shard_index) + " not below n = " +
                           std::to_string(info.n));
    if (symbols > 0xFFFFFFFFull) throw SizeMismatch("payload too long for a shard");
    if (esc.size() > 65535)
        throw TooManyEscapes(std::to_string(esc.size()) + " escaped symbols in one shard, limit is 65535");
    std::vector<uint8_t> out;
    out.reserve(kShardHeader + 4 * esc.size() + 2 * symbols);
    out.insert(out.end(), kShardMagic, kShardMagic + 4);
    BeOut w{out};
    w.u(kVersion, 1);
    w.u(info.chunk_id, 8);
    w.u(info.k, 2);
    w.u(n_wire(info.n), 2);
    w.u(info.shard_index, 2);
    w.u(info.systematic ? kSystematicFlag : 0, 1);
    w.u(symbols, 4);
    w.u(esc.size(), 2);
    for (uint64_t e : esc) w.u(e, 4);
    return out;
}

ParsedShard parse_shard(std::span<const std::uint8_t> bytes) {
    BeIn r{bytes};
    r.magic(kShardMagic);
    if (const uint64_t v = r.u(1); v != kVersion)
        throw BadVersion("shard version " + std::to_string(v) + ", expected " + std::to_string(kVersion));
    ReadShard s;
    s.info.chunk_id = r.u(8);
    s.info.k = uint32_t(r.u(2));
    s.info.n = n_unwire(r.u(2));
    s.info.shard_index = uint32_t(r.u(2));
    const uint64_t flags = r.u(1);
    if (flags & ~uint64_t(kSystematicFlag)) throw MalformedHeader("unknown flag bits set: " + std::to_string(flags));
    s.info.systematic = flags & kSystematicFlag;
    const uint32_t symbols = uint32_t(r.u(4));
    const uint32_t nesc = uint32_t(r.u(2));
    if (s.info.k == 0) throw MalformedHeader("shard header has k = 0");
    if (s.info.n < s.info.k)
        throw MalformedHeader("shard header has n = " + std::to_string(s.info.n) + " below k = " +
                              std::to_string(s.info.k));
    if (s.info.shard_index >= s.info.n)
        throw MalformedHeader("shard index " + std::to_string(s.info.shard_index) + " not below n = " +
                              std::to_string(s.info.n));
    std::vector<uint32_t> esc(nesc);
    for (auto& e : esc) e = uint32_t(r.u(4));
    for (size_t i = 0; i < esc.size(); ++i) {
        if (esc[i] >= symbols)
            throw MalformedEscapes("escape position " + std::to_string(esc[i]) + " not below payload size " +
                                   std::to_string(symbols));
        if (i && esc[i] <= esc[i - 1]) throw MalformedEscapes("escape positions not strictly increasing");
    }
    r.need(size_t(2) * symbols);
    const size_t at = r.at;
    r.at += size_t(2) * symbols;
    if (r.at != bytes.size())
        throw MalformedHeader(std::to_string(bytes.size() - r.at) + " trailing bytes after the payload");
    for (uint32_t e : esc)
        if (bytes[at + 2 * size_t(e)] | bytes[at + 2 * size_t(e) + 1])
            throw MalformedEscapes("escape at position " + std::to_string(e) + " points at a nonzero word");
    return ParsedShard{s.info, symbols, std::move(esc), at};
}
}  // namespace detail

std::vector<std::uint8_t> write_shard(const ShardInfo& info, std::span<const Fe> payload) {
    std::vector<uint16_t> words;
    std::vector<uint64_t> esc;
    if (info.k >= 1 && info.k <= 65535 && info.n >= info.k && info.n <= 65536 && info.shard_index < info.n)
        split(payload.data(), payload.size(), words, esc);  // SizeMismatch on values above 65536
    std::vector<uint8_t> out = detail::shard_header(info, payload.size(), esc);  // header checks first
    const size_t at = out.size();
    out.resize(at + 2 * words.size());
    words_to_be(words, out.data() + at);
    return out;
}

ReadShard read_shard(std::span<const std::uint8_t> bytes) {
    detail::ParsedShard p = detail::parse_shard(bytes);
    ReadShard s;
    s.info = p.info;
    const std::vector<uint16_t> words = be_to_words(bytes.data() + p.payload_offset, p.symbols);
    s.payload.assign(words.begin(), words.end());
    for (uint32_t e : p.escapes) s.payload[e] = 65536;
    return s;
}

std::vector<std::uint8_t> write_manifest(const ChunkManifest& m) {
    if (m.k < 1 || m.k > 65535) throw SizeMismatch("manifest k must be in [1, 65535], got " + std::to_string(m.k));
    if (m.n < m.k || m.n > 65536) throw SizeMismatch("manifest n must be in [k, 65536], got " + std::to_string(m.n));
    if (m.original_length > uint64_t(m.stripes) * m.k * 2)
        throw LengthMismatch("manifest length " + std::to_string(m.original_length) + " exceeds stripe capacity");
    std::vector<uint8_t> out;
    out.reserve(kManifestBytes);
    out.insert(out.end(), kManifestMagic, kManifestMagic + 4);
    BeOut w{out};
    w.u(kVersion, 1);
    w.u(m.chunk_id, 8);
    w.u(m.original_length, 8);
    w.u(m.k, 2);
    w.u(n_wire(m.n), 2);
    w.u(m.stripes, 4);
    w.u(m.systematic ? kSystematicFlag : 0, 1);
    return out;
}

ChunkManifest read_manifest(std::span<const std::uint8_t> bytes) {
    BeIn r{bytes};
    r.magic(kManifestMagic);
    if (const uint64_t v = r.u(1); v != kVersion)
        throw BadVersion("manifest version " + std::to_string(v) + ", expected " + std::to_string(kVersion));
    ChunkManifest m;
    m.chunk_id = r.u(8);
    m.original_length = r.u(8);
    m.k = uint32_t(r.u(2));
    m.n = n_unwire(r.u(2));
    m.stripes = uint32_t(r.u(4));
    const uint64_t flags = r.u(1);
    if (flags & ~uint64_t(kSystematicFlag)) throw MalformedHeader("unknown flag bits set: " + std::to_string(flags));
    m.systematic = flags & kSystematicFlag;
    if (r.at != bytes.size())
        throw MalformedHeader(std::to_string(bytes.size() - r.at) + " trailing bytes after the manifest");
    if (m.k == 0) throw MalformedHeader("manifest has k = 0");
    if (m.n < m.k) throw MalformedHeader("manifest has n below k");
    if (m.original_length > uint64_t(m.stripes) * m.k * 2)
        throw MalformedHeader("manifest length exceeds stripe capacity");
    return m;
}

std::string shard_filename(std::uint64_t chunk_id, std::uint32_t shard_index) {
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%016llx.%u.fnt", static_cast<unsigned long long>(chunk_id), shard_index);
    return buf;
}

std::string manifest_filename(std::uint64_t chunk_id) {
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%016llx.manifest.fnt", static_cast<unsigned long long>(chunk_id));
    return buf;
}

}  // namespace shardio
}  // namespace fntrs
