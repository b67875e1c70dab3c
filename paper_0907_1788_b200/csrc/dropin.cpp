// dropin.cpp -- the reference's C++ codec API (include/fntrs/codec.hpp) over
// the C ABI (include/fntrs_gpu.h). Host work here is the reference's own
// host logic -- argument validation, sorting the received symbols
// (proj/src/codec.cpp:32-48), the 16-entry decode-plan LRU
// (proj/src/interp.cpp:70-101) -- plus marshalling Fe <-> uint16 + escapes.
// All arithmetic runs on the GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "fntrs/codec.hpp"
#include "fntrs/instrument.hpp"
#include "fntrs/interp.hpp"
#include "fntrs/transform.hpp"
#include "fntrs_gpu.h"
#include "dropin_shared.h"
#include "fntrs/poly.hpp"

namespace fntrs {

// ---- instrumentation (instrument.hpp): counters and the per-thread scope chain
namespace {
thread_local FntScope* g_scope = nullptr;
std::size_t size_bucket(std::size_t size) noexcept {  // ceil(log2 size), capped at 2^16
    std::size_t lg = 0;
    while (lg < 16 && (std::size_t{1} << lg) < size) ++lg;
    return lg;
}
}  // namespace
void FntCounter::record(std::size_t size) noexcept { ++by_log2_[size_bucket(size)]; }
std::uint64_t FntCounter::count(std::size_t size) const noexcept { return by_log2_[size_bucket(size)]; }
std::uint64_t FntCounter::total() const noexcept {
    std::uint64_t sum = 0;
    for (std::uint64_t c : by_log2_) sum += c;
    return sum;
}
double FntCounter::equivalents(std::size_t base) const noexcept {
    double work = 0.0;
    for (std::size_t lg = 0; lg < by_log2_.size(); ++lg) work += double(by_log2_[lg]) * double(std::size_t{1} << lg);
    return work / double(base);
}
void FntCounter::merge(const FntCounter& other) noexcept {
    for (std::size_t lg = 0; lg < by_log2_.size(); ++lg) by_log2_[lg] += other.by_log2_[lg];
}
std::map<std::size_t, std::uint64_t> FntCounter::snapshot() const {
    std::map<std::size_t, std::uint64_t> out;
    for (std::size_t lg = 0; lg < by_log2_.size(); ++lg)
        if (by_log2_[lg]) out[std::size_t{1} << lg] = by_log2_[lg];
    return out;
}
FntScope::FntScope(FntCounter& counter) : counter_(counter), outer_(g_scope) { g_scope = this; }
FntScope::~FntScope() { g_scope = outer_; }
void note_fnt_execution(std::size_t size) noexcept {
    for (FntScope* s = g_scope; s; s = s->outer_) s->counter_.record(size);
}

void throw_status(int status, const std::string& msg) {
    switch (status) {
        case FNTRS_E_ZERO_INVERSE: throw ZeroInverse(msg);
        case FNTRS_E_INVALID_TRANSFORM_SIZE: throw InvalidTransformSize(msg);
        case FNTRS_E_SIZE_MISMATCH: throw SizeMismatch(msg);
        case FNTRS_E_PRODUCT_TOO_LARGE: throw ProductTooLarge(msg);
        case FNTRS_E_DUPLICATE_POINT: throw DuplicatePoint(msg);
        case FNTRS_E_DUPLICATE_POSITION: throw DuplicatePosition(msg);
        case FNTRS_E_POSITION_OUT_OF_RANGE: throw PositionOutOfRange(msg);
        case FNTRS_E_TOO_FEW_POSITIONS: throw TooFewPositions(msg);
        case FNTRS_E_NOT_ENOUGH_SYMBOLS: throw NotEnoughSymbols(msg);
        case FNTRS_E_TOO_MANY_ESCAPES: throw TooManyEscapes(msg);
        case FNTRS_E_BAD_MAGIC: throw BadMagic(msg);
        case FNTRS_E_BAD_VERSION: throw BadVersion(msg);
        case FNTRS_E_TRUNCATED_SHARD: throw TruncatedShard(msg);
        case FNTRS_E_MALFORMED_ESCAPES: throw MalformedEscapes(msg);
        case FNTRS_E_MALFORMED_HEADER: throw MalformedHeader(msg);
        case FNTRS_E_LENGTH_MISMATCH: throw LengthMismatch(msg);
        case FNTRS_E_NOT_ENOUGH_SHARDS: throw NotEnoughShards(msg);
        default: throw Error(msg);
    }
}

namespace dropin {
Shared& shared() {
    // never destroyed: releasing device state from a static destructor can run
    // after the CUDA runtime has shut down; the process exit frees it all
    static Shared* s = new Shared;
    return *s;
}
}  // namespace dropin
using namespace dropin;

namespace gpu {
void set_device(int device) {
    Shared& S = shared();
    std::lock_guard<std::mutex> lock(S.mu);
    if (S.ctx && S.device != device) {
        for (auto& e : S.lru) fntrs_gpu_plans_destroy(e.second);
        S.lru.clear();
        if (S.dbuf) cudaFree(S.dbuf);
        S.dbuf = nullptr;
        S.dbuf_bytes = 0;
        if (S.zero_pattern) cudaFree(S.zero_pattern);
        S.zero_pattern = nullptr;
        if (S.stream) cudaStreamDestroy(S.stream);
        S.stream = nullptr;
        fntrs_gpu_destroy(S.ctx);
        S.ctx = nullptr;
    }
    S.device = device;
}
}  // namespace gpu

namespace codec {

CodeParams CodeParams::make(std::uint32_t k, std::uint32_t n, bool systematic) {
    uint32_t nd = 0;
    if (fntrs_gpu_code_params(k, n, &nd) != FNTRS_OK)
        throw SizeMismatch("code parameters need 1 <= k <= n <= 65536, got k = " + std::to_string(k) +
                           ", n = " + std::to_string(n));
    CodeParams p;
    p.k = k;
    p.n = n;
    p.n_domain = nd;
    p.systematic = systematic;
    return p;
}

namespace {
std::vector<Fe> encode_one(const CodeParams& params, std::span<const Fe> source, bool systematic) {
    if (source.size() != params.k)
        throw SizeMismatch("encode: got " + std::to_string(source.size()) + " source symbols for k = " +
                           std::to_string(params.k));
    Shared& S = shared();
    std::lock_guard<std::mutex> lock(S.mu);
    S.ensure();
    std::vector<uint16_t> words;
    std::vector<uint64_t> esc;
    split(source.data(), source.size(), words, esc);
    auto fn = systematic ? fntrs_gpu_encode_systematic : fntrs_gpu_encode;
    auto out = run(S, words, esc, params.n,
                   [&](const uint16_t* din, const uint64_t* die, uint64_t nie, uint16_t* dout, uint64_t* doe,
                       uint64_t cap, uint64_t* dcnt) {
                       S.check(fn(S.ctx, params.k, params.n, 1, 1, din, die, nie, dout, doe, cap, dcnt, S.stream));
                   });
    S.note_transforms();
    return out;
}

// sorted_received (codec.cpp:32-48): range check, sort, duplicates, count
Codeword sorted_received(const CodeParams& params, const Codeword& received) {
    for (const Symbol& s : received)
        if (s.position >= params.n)
            throw PositionOutOfRange("received position " + std::to_string(s.position) + " not below n = " +
                                     std::to_string(params.n));
    Codeword sorted(received);
    std::sort(sorted.begin(), sorted.end(), [](const Symbol& a, const Symbol& b) { return a.position < b.position; });
    for (size_t i = 1; i < sorted.size(); ++i)
        if (sorted[i].position == sorted[i - 1].position)
            throw DuplicatePosition("received position " + std::to_string(sorted[i].position) + " repeats");
    if (sorted.size() < params.k)
        throw NotEnoughSymbols("have " + std::to_string(sorted.size()) + " symbols, need " +
                               std::to_string(params.k));
    return sorted;
}

// Decode one codeword from the kp lowest received symbols.
std::vector<Fe> decode_one(const CodeParams& params, const Codeword& sorted, uint32_t kp, bool systematic) {
    std::vector<uint32_t> pos(kp);
    std::vector<Fe> vals(kp);
    for (uint32_t i = 0; i < kp; ++i) {
        pos[i] = sorted[i].position;
        vals[i] = sorted[i].value;
    }
    Shared& S = shared();
    std::lock_guard<std::mutex> lock(S.mu);
    S.ensure();
    fntrs_plans* plan = S.plan_for(params.k, params.n, pos);
    std::vector<uint16_t> words;
    std::vector<uint64_t> esc;
    split(vals.data(), vals.size(), words, esc);
    auto fn = systematic ? fntrs_gpu_decode_systematic : fntrs_gpu_decode;
    std::vector<Fe> out = run(S, words, esc, params.k,
                              [&](const uint16_t* din, const uint64_t* die, uint64_t nie, uint16_t* dout,
                                  uint64_t* doe, uint64_t cap, uint64_t* dcnt) {
                                  S.check(fn(S.ctx, plan, 1, 1, S.zero_pattern, din, die, nie, dout, doe, cap, dcnt,
                                             S.stream));
                              });
    S.note_transforms();
    return out;
}
}  // namespace

std::vector<Fe> encode_nonsystematic(const CodeParams& params, std::span<const Fe> source) {
    return encode_one(params, source, false);
}

std::vector<Fe> decode_nonsystematic(const CodeParams& params, const Codeword& received, Path) {
    Codeword sorted = sorted_received(params, received);
    const bool full = params.n == next_pow2(params.n) && sorted.size() == params.n;  // codec.cpp:137-144
    return decode_one(params, sorted, full ? params.n : params.k, false);  // else the k lowest positions
}

std::vector<Fe> encode_systematic(const CodeParams& params, std::span<const Fe> source, Path) {
    return encode_one(params, source, true);
}

std::vector<Fe> encode_systematic_direct(const CodeParams& params, std::span<const Fe> source) {
    return encode_one(params, source, true);
}

std::vector<Fe> encode_systematic_intermediate_direct(const CodeParams& params, std::span<const Fe> source) {
    return encode_one(params, source, true);
}

std::vector<Fe> decode_direct(const CodeParams& params, const Codeword& received) {  // codec.cpp:255-258
    return params.systematic ? decode_systematic(params, received, Path::Direct)
                             : decode_nonsystematic(params, received, Path::Direct);
}

std::vector<Fe> decode_systematic(const CodeParams& params, const Codeword& received, Path) {
    // interpolate the k lowest, evaluate at 0..k-1; when those are 0..k-1 the
    // result is the received values themselves (systematic_prefix_present,
    // codec.cpp:167-171: a copy, no transforms -- the kernels would reproduce
    // the same values)
    Codeword sorted = sorted_received(params, received);
    bool prefix = true;
    for (uint32_t i = 0; i < params.k && prefix; ++i) prefix = sorted[i].position == i;
    if (prefix) {
        Shared& S = shared();
        std::lock_guard<std::mutex> lock(S.mu);
        S.ensure();  // no device, no codec: fail loudly like every other call
        std::vector<Fe> out(params.k);
        for (uint32_t i = 0; i < params.k; ++i) out[i] = sorted[i].value;
        return out;
    }
    return decode_one(params, sorted, params.k, true);
}

}  // namespace codec

// ---- transform API (transform.hpp) ---------------------------------------
namespace {
bool pow2_domain(uint32_t n) { return n >= 1 && n <= 65536 && (n & (n - 1)) == 0; }

uint32_t bitrev(uint32_t i, uint32_t n) {
    uint32_t r = 0;
    for (uint32_t b = 1; b < n; b <<= 1, i >>= 1) r = (r << 1) | (i & 1u);
    return r;
}

// one vector through fntrs_gpu_fnt (mode 0 forward, 1 inverse, 2 unscaled inverse)
std::vector<Fe> fnt_device(uint32_t n, const Fe* in, int mode) {
    Shared& S = shared();
    std::lock_guard<std::mutex> lock(S.mu);
    S.ensure();
    const size_t bytes = (size_t(n) * 4 + 255) / 256 * 256;
    auto* d = static_cast<uint32_t*>(S.scratch(2 * bytes));
    cudaMemcpyAsync(d, in, size_t(n) * 4, cudaMemcpyHostToDevice, S.stream);
    S.check(fntrs_gpu_fnt(S.ctx, n, mode, 1, d, d + bytes / 4, S.stream));
    std::vector<Fe> out(n);
    cudaMemcpyAsync(out.data(), d + bytes / 4, size_t(n) * 4, cudaMemcpyDeviceToHost, S.stream);
    S.sync();
    S.note_transforms();
    return out;
}
}  // namespace

TransformPlan::TransformPlan(std::uint32_t n) : size(n) {
    if (!pow2_domain(n)) throw InvalidTransformSize("transform size must be a power of two in [1, 65536], got " +
                                                    std::to_string(n));
    root = gf::root_of_unity(n);
    inverse_root = gf::root_of_unity(n, true);
    size_inverse = gf::inv(n % gf::prime);
    // the reference's tables (transform.cpp:31-63), filled on the device
    const size_t h = n / 2, st = n > 1 ? n - 1 : 0;
    twiddles.resize(h);
    inverse_twiddles.resize(h);
    bit_reversal.resize(n);
    stage_twiddles.resize(st);
    stage_inverse_twiddles.resize(st);
    Shared& S = shared();
    std::lock_guard<std::mutex> lock(S.mu);
    S.ensure();
    DevBuf d((2 * h + n + 2 * st + 1) * 4, S.stream);
    uint32_t* p = d.as<uint32_t>();
    S.check(fntrs_gpu_transform_tables(S.ctx, n, p, p + h, p + 2 * h, p + 2 * h + n, p + 2 * h + n + st, S.stream));
    download(S, twiddles.data(), d, h, 0);
    download(S, inverse_twiddles.data(), d, h, h);
    download(S, bit_reversal.data(), d, n, 2 * h);
    download(S, stage_twiddles.data(), d, st, 2 * h + n);
    download(S, stage_inverse_twiddles.data(), d, st, 2 * h + n + st);
    S.sync();
}

std::vector<Fe> naive_dft(Fe root, std::span<const Fe> a, bool inverse) {  // transform.cpp:325-343
    const size_t n = a.size();
    std::vector<Fe> out(n);
    Shared& S = shared();
    std::lock_guard<std::mutex> lock(S.mu);
    S.ensure();
    if (!n) return out;
    DevBuf d(2 * n * 4, S.stream);
    upload(S, d, a.data(), n);
    S.check(fntrs_gpu_naive_dft(S.ctx, root, inverse ? 1 : 0, uint32_t(n), d.as<uint32_t>(), d.as<uint32_t>() + n,
                                S.stream));
    download(S, out.data(), d, n, n);
    S.sync();
    return out;
}

const TransformPlan& plan_for(std::uint32_t n) {
    static std::mutex mu;
    static std::array<std::unique_ptr<TransformPlan>, 17> plans;
    if (!pow2_domain(n)) throw InvalidTransformSize("transform size must be a power of two in [1, 65536], got " +
                                                    std::to_string(n));
    uint32_t lg = 0;
    while ((1u << lg) < n) ++lg;
    std::lock_guard<std::mutex> lock(mu);
    if (!plans[lg]) plans[lg] = std::make_unique<TransformPlan>(n);
    return *plans[lg];
}

std::vector<Fe> fnt_forward(const TransformPlan& plan, std::span<const Fe> a) {
    if (a.size() != plan.size) throw SizeMismatch("transform input has " + std::to_string(a.size()) +
                                                  " values for size " + std::to_string(plan.size));
    return fnt_device(plan.size, a.data(), 0);
}

std::vector<Fe> fnt_inverse(const TransformPlan& plan, std::span<const Fe> a) {
    if (a.size() != plan.size) throw SizeMismatch("transform input has " + std::to_string(a.size()) +
                                                  " values for size " + std::to_string(plan.size));
    return fnt_device(plan.size, a.data(), 1);
}

void dif_forward(const TransformPlan& plan, std::span<Fe> data) {
    if (data.size() != plan.size) throw SizeMismatch("transform input length mismatch");
    auto y = fnt_device(plan.size, data.data(), 0);  // natural order
    for (uint32_t i = 0; i < plan.size; ++i) data[i] = y[bitrev(i, plan.size)];
}

void dit_inverse_unscaled(const TransformPlan& plan, std::span<Fe> data) {
    if (data.size() != plan.size) throw SizeMismatch("transform input length mismatch");
    std::vector<Fe> x(plan.size);
    for (uint32_t i = 0; i < plan.size; ++i) x[bitrev(i, plan.size)] = data[i];  // to natural order
    auto y = fnt_device(plan.size, x.data(), 2);
    std::copy(y.begin(), y.end(), data.begin());
}

// ---- plan-level API (interp.hpp) ------------------------------------------
namespace interp {

namespace {
std::vector<Fe> points_of(uint32_t n, const std::vector<uint32_t>& positions) {
    const Fe r = gf::root_of_unity(n);
    std::vector<Fe> xs(positions.size());
    for (size_t i = 0; i < xs.size(); ++i) xs[i] = gf::pow(r, positions[i]);
    return xs;
}
}  // namespace

poly::Poly lagrange_oracle(std::span<const std::pair<Fe, Fe>> points) {  // interp.cpp:139-171
    const size_t k = points.size();
    std::vector<Fe> xs(k), vs(k);
    for (size_t i = 0; i < k; ++i) {
        xs[i] = points[i].first;
        vs[i] = points[i].second;
    }
    {
        std::vector<Fe> sorted(xs);
        std::sort(sorted.begin(), sorted.end());
        auto dup = std::adjacent_find(sorted.begin(), sorted.end());
        if (dup != sorted.end()) throw DuplicatePoint("interpolation point " + std::to_string(*dup) + " repeats");
    }
    Shared& S = shared();
    std::lock_guard<std::mutex> lock(S.mu);
    S.ensure();
    if (k == 0) return {};
    DevBuf d(3 * k * 4, S.stream);
    upload(S, d, xs.data(), k);
    uint32_t* p = d.as<uint32_t>();
    if (cudaMemcpyAsync(p + k, vs.data(), k * 4, cudaMemcpyHostToDevice, S.stream) != cudaSuccess)
        throw Error("fntrs: host-to-device copy failed");
    S.check(fntrs_gpu_lagrange(S.ctx, uint32_t(k), p, p + k, p + 2 * k, S.stream));
    poly::Poly out(k);
    download(S, out.data(), d, k, 2 * k);
    S.sync();
    poly::normalize(out);
    return out;
}

DecodePlan build_plan(std::uint32_t n, std::span<const std::uint32_t> positions) {  // interp.cpp:23-68 checks
    if (positions.empty()) throw TooFewPositions("no positions to build a plan from");
    if (!pow2_domain(n)) throw InvalidTransformSize("plan domain must be a power of two in [1, 65536]");
    for (uint32_t z : positions)
        if (z >= n)
            throw PositionOutOfRange("position " + std::to_string(z) + " not below domain size " + std::to_string(n));
    {
        std::vector<uint32_t> sorted(positions.begin(), positions.end());
        std::sort(sorted.begin(), sorted.end());
        auto dup = std::adjacent_find(sorted.begin(), sorted.end());
        if (dup != sorted.end()) throw DuplicatePosition("position " + std::to_string(*dup) + " repeats");
    }
    const uint32_t k = uint32_t(positions.size());
    DecodePlan plan;
    plan.n = n;
    plan.k = k;
    plan.positions.assign(positions.begin(), positions.end());
    Shared& S = shared();
    std::lock_guard<std::mutex> lock(S.mu);
    S.ensure();
    fntrs_plans* pl = nullptr;
    S.check(fntrs_gpu_plans_create(S.ctx, k, n, k, 1, plan.positions.data(), &pl, S.stream));
    plan.device = std::shared_ptr<const void>(pl, [](const void* p) {
        fntrs_gpu_plans_destroy(static_cast<fntrs_plans*>(const_cast<void*>(p)));
    });
    const uint32_t m = 2ull * k > 65536ull ? 65536u : next_pow2(2 * k);
    plan.aprime_at_x_inv.assign(k, 0);
    std::vector<Fe> afnt(m);
    uint32_t ps = 0;
    S.sync();
    S.check(fntrs_gpu_plans_export(S.ctx, pl, 0, nullptr, plan.aprime_at_x_inv.data(), &ps, afnt.data()));
    plan.product_size = ps;
    afnt.resize(ps);
    plan.a_fnt = std::move(afnt);
    plan.a_tree = tree_on_device(S, points_of(n, plan.positions));  // x_i = r^(z_i), interp.cpp:30-35
    S.note_transforms();
    return plan;
}

std::shared_ptr<const DecodePlan> plan_for(std::uint32_t n, std::span<const std::uint32_t> positions) {
    static std::mutex mu;  // interp.cpp:70-101: LRU of 16, canonical ascending positions
    static std::list<std::pair<std::vector<uint32_t>, std::shared_ptr<const DecodePlan>>> lru;
    std::vector<uint32_t> key(positions.begin(), positions.end());
    std::sort(key.begin(), key.end());
    key.push_back(n);
    {
        std::lock_guard<std::mutex> lock(mu);
        for (auto it = lru.begin(); it != lru.end(); ++it)
            if (it->first == key) {
                lru.splice(lru.begin(), lru, it);
                return lru.front().second;
            }
    }
    auto plan = std::make_shared<const DecodePlan>(build_plan(n, std::span<const uint32_t>(key.data(), key.size() - 1)));
    std::lock_guard<std::mutex> lock(mu);
    lru.emplace_front(key, plan);
    if (lru.size() > 16) lru.pop_back();
    return plan;
}

poly::Poly interpolate(const DecodePlan& plan, std::span<const Fe> values) {
    if (values.size() != plan.k)
        throw SizeMismatch("interpolate: got " + std::to_string(values.size()) + " values for " +
                           std::to_string(plan.k) + " positions");
    auto* pl = static_cast<fntrs_plans*>(const_cast<void*>(plan.device.get()));
    if (!pl) throw Error("interpolate: plan has no device state");
    Shared& S = shared();
    std::lock_guard<std::mutex> lock(S.mu);
    S.ensure();
    std::vector<uint16_t> words;
    std::vector<uint64_t> esc;
    split(values.data(), values.size(), words, esc);
    poly::Poly p = run(S, words, esc, plan.k,
                       [&](const uint16_t* din, const uint64_t* die, uint64_t nie, uint16_t* dout, uint64_t* doe,
                           uint64_t cap, uint64_t* dcnt) {
                           S.check(fntrs_gpu_decode(S.ctx, pl, 1, 1, S.zero_pattern, din, die, nie, dout, doe, cap,
                                                    dcnt, S.stream));
                       });
    S.note_transforms();
    while (!p.empty() && p.back() == 0) p.pop_back();  // poly::normalize
    return p;
}

}  // namespace interp
}  // namespace fntrs
