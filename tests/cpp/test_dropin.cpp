// tests/cpp/test_dropin.cpp -- the reference's own codec test cases, run
// against the drop-in C++ API (include/fntrs/codec.hpp) on the GPU.
// Cases follow /root/reference/proj/tests/test_codec.cpp (file:line in each
// section); values are the reference's frozen golden vectors. Built by
// `make cpptest`, run by tests/test_gpu_parity.py::test_cpp_dropin (gpu).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <random>
#include <atomic>
#include <thread>
#include <vector>

#include "fntrs/codec.hpp"
#include "fntrs/instrument.hpp"
#include "fntrs/geom.hpp"
#include "fntrs/interp.hpp"
#include "fntrs/poly.hpp"
#include "fntrs/shardio.hpp"
#include "fntrs/transform.hpp"

using namespace fntrs;
using namespace fntrs::codec;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                        \
    do {                                                                   \
        if (cond) {                                                        \
            ++g_pass;                                                      \
        } else {                                                           \
            ++g_fail;                                                      \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                  \
    } while (0)

template <typename E, typename F>
static bool throws_as(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static std::vector<Fe> random_source(uint32_t k, uint32_t seed) {
    std::mt19937 rng(seed);
    std::uniform_int_distribution<uint32_t> d(0, 65536);
    std::vector<Fe> v(k);
    for (auto& x : v) x = d(rng);
    return v;
}

static Codeword take(const std::vector<Fe>& enc, const std::vector<uint32_t>& pos) {
    Codeword c;
    for (uint32_t p : pos) c.push_back({p, enc[p]});
    return c;
}

static void for_each_subset(uint32_t n, uint32_t s, const std::function<void(const std::vector<uint32_t>&)>& fn) {
    std::vector<uint32_t> idx(s);
    for (uint32_t i = 0; i < s; ++i) idx[i] = i;
    for (;;) {
        fn(idx);
        int i = int(s) - 1;
        while (i >= 0 && idx[i] == n - s + uint32_t(i)) --i;
        if (i < 0) return;
        ++idx[i];
        for (uint32_t j = uint32_t(i) + 1; j < s; ++j) idx[j] = idx[j - 1] + 1;
    }
}

int main() {
    // CodeParams (test_codec.cpp:60-70)
    {
        auto p = CodeParams::make(3, 6);
        CHECK(p.k == 3 && p.n == 6 && p.n_domain == 8);
        CHECK(CodeParams::make(16, 16).n_domain == 16);
        CHECK(CodeParams::make(1, 65536).n_domain == 65536);
        CHECK(throws_as<SizeMismatch>([] { CodeParams::make(0, 4); }));
        CHECK(throws_as<SizeMismatch>([] { CodeParams::make(5, 4); }));
        CHECK(throws_as<SizeMismatch>([] { CodeParams::make(1, 65537); }));
    }
    // non-systematic encode basics (test_codec.cpp:72-84)
    {
        auto p15 = CodeParams::make(1, 5, false);
        CHECK(encode_nonsystematic(p15, std::vector<Fe>{77}) == (std::vector<Fe>{77, 77, 77, 77, 77}));
        auto p24 = CodeParams::make(2, 4, false);
        CHECK(encode_nonsystematic(p24, std::vector<Fe>{5, 7}) == (std::vector<Fe>{12, 63750, 65535, 1797}));
        CHECK(throws_as<SizeMismatch>([&] { encode_nonsystematic(p24, std::vector<Fe>{1}); }));
    }
    // rate-1 code (test_codec.cpp:86-94): decode of all symbols inverts
    {
        auto p = CodeParams::make(8, 8, false);
        auto src = random_source(8, 1);
        auto enc = encode_nonsystematic(p, src);
        CHECK(decode_nonsystematic(p, take(enc, {0, 1, 2, 3, 4, 5, 6, 7})) == src);
        // size-8 frozen transform (test_transform.cpp:51-57): k = n = 8 encode is fnt_forward
        CHECK(encode_nonsystematic(p, std::vector<Fe>{1, 2, 3, 4, 5, 6, 7, 8}) ==
              (std::vector<Fe>{36, 50109, 1020, 48061, 65533, 17468, 64509, 15420}));
    }
    // frozen decode (test_codec.cpp:96-102)
    {
        auto p = CodeParams::make(2, 4, false);
        Codeword rx{{0, 12}, {2, 65535}};
        CHECK(decode_nonsystematic(p, rx) == (std::vector<Fe>{5, 7}));
        CHECK(decode_nonsystematic(p, rx, Path::Fast) == (std::vector<Fe>{5, 7}));
    }
    // validation (test_codec.cpp:104-112)
    {
        auto p = CodeParams::make(2, 4, false);
        CHECK(throws_as<NotEnoughSymbols>([&] { decode_nonsystematic(p, Codeword{{0, 1}}); }));
        CHECK(throws_as<DuplicatePosition>([&] { decode_nonsystematic(p, Codeword{{1, 5}, {1, 6}}); }));
        CHECK(throws_as<PositionOutOfRange>([&] { decode_nonsystematic(p, Codeword{{0, 5}, {4, 6}}); }));
    }
    // MDS: every erasure pattern decodes (test_codec.cpp:192-224)
    {
        const std::pair<uint32_t, uint32_t> cases[] = {{4, 2}, {8, 4}, {8, 5}, {16, 12}};
        for (auto [n, k] : cases) {
            auto p = CodeParams::make(k, n, false);
            auto src = random_source(k, n * 31 + k);
            auto enc = encode_nonsystematic(p, src);
            uint64_t patterns = 0, ok = 0;
            for (uint32_t s = k; s <= n; ++s)
                for_each_subset(n, s, [&](const std::vector<uint32_t>& keep) {
                    ++patterns;
                    ok += decode_nonsystematic(p, take(enc, keep), Path::Fast) == src;
                });
            uint64_t expected = 0;
            for (uint32_t s = k; s <= n; ++s) {
                uint64_t c = 1;
                for (uint32_t i = 0; i < s; ++i) c = c * (n - i) / (i + 1);
                expected += c;
            }
            CHECK(patterns == expected);
            CHECK(ok == patterns);
            std::printf("MDS n=%u k=%u: %llu/%llu patterns decode\n", n, k, (unsigned long long)ok,
                        (unsigned long long)patterns);
        }
    }
    // received order is irrelevant (test_codec.cpp:226-236, non-systematic here)
    {
        auto p = CodeParams::make(5, 11, false);
        auto src = random_source(5, 17);
        auto enc = encode_nonsystematic(p, src);
        Codeword rx = take(enc, {9, 2, 7, 4, 10, 3});
        std::mt19937 rng(18);
        for (int i = 0; i < 10; ++i) {
            std::shuffle(rx.begin(), rx.end(), rng);
            CHECK(decode_nonsystematic(p, rx) == src);
        }
    }
    // k lowest positions win (test_codec.cpp:238-247)
    {
        auto p = CodeParams::make(3, 9, false);
        auto src = random_source(3, 19);
        auto enc = encode_nonsystematic(p, src);
        auto tampered = enc;
        tampered[8] = gf::add(tampered[8], 1);
        CHECK(decode_nonsystematic(p, take(tampered, {1, 3, 5, 8})) == src);
    }
    // sources holding the top field value (test_codec.cpp:333-339, non-systematic)
    {
        auto p = CodeParams::make(3, 7, false);
        std::vector<Fe> src{65536, 65536, 65536};
        auto enc = encode_nonsystematic(p, src);
        CHECK(decode_nonsystematic(p, take(enc, {2, 4, 6})) == src);
    }
    // systematic encode carries the source verbatim (test_codec.cpp:112-124)
    {
        const std::pair<uint32_t, uint32_t> cases[] = {{1, 6}, {2, 4}, {4, 8}, {5, 13}, {300, 700}};
        for (auto [k, n] : cases) {
            auto params = CodeParams::make(k, n);
            auto src = random_source(k, 100 + k);
            for (Path path : {Path::Fast, Path::Direct}) {
                auto enc = encode_systematic(params, src, path);
                CHECK(enc.size() == n);
                CHECK(std::equal(src.begin(), src.end(), enc.begin()));
            }
        }
    }
    // all systematic encoder variants agree (test_codec.cpp:138-154)
    {
        std::mt19937 rng(7);
        for (int trial = 0; trial < 20; ++trial) {
            uint32_t k = std::uniform_int_distribution<uint32_t>(1, 64)(rng);
            uint32_t n = std::uniform_int_distribution<uint32_t>(k, 150)(rng);
            auto params = CodeParams::make(k, n);
            auto src = random_source(k, 200 + trial);
            auto fast = encode_systematic(params, src, Path::Fast);
            CHECK(encode_systematic_direct(params, src) == fast);
            CHECK(encode_systematic_intermediate_direct(params, src) == fast);
            CHECK(encode_systematic(params, src, Path::Auto) == fast);
            auto enc = encode_nonsystematic(CodeParams::make(k, n, false), src);
            Codeword rx;
            for (uint32_t i = n - k; i < n; ++i) rx.push_back({i, enc[i]});
            CHECK(decode_direct(CodeParams::make(k, n, false), rx) == src);
        }
    }
    // systematic encode frozen examples (test_codec.cpp:126-136)
    {
        CHECK(encode_systematic(CodeParams::make(2, 4), std::vector<Fe>{5, 7}) ==
              (std::vector<Fe>{5, 7, 65032, 65030}));
        CHECK(encode_systematic(CodeParams::make(4, 8), std::vector<Fe>{100, 200, 300, 400}) ==
              (std::vector<Fe>{100, 200, 300, 400, 33256, 17912, 53593, 3200}));
        CHECK(encode_systematic(CodeParams::make(1, 6), std::vector<Fe>{9}) == std::vector<Fe>(6, 9));
    }
    // systematic decode shortcuts and reconstructions (test_codec.cpp:164-190)
    {
        auto params = CodeParams::make(4, 8);
        std::vector<Fe> src{100, 200, 300, 400};
        auto enc = encode_systematic(params, src);
        CHECK(decode_systematic(params, take(enc, {0, 1, 2, 3, 6})) == src);
        CHECK(decode_systematic(params, take(enc, {2, 3, 4, 5, 6, 7}), Path::Fast) == src);
        CHECK(decode_systematic(params, take(enc, {2, 3, 4, 5, 6, 7}), Path::Direct) == src);
        CHECK(throws_as<NotEnoughSymbols>([&] { decode_systematic(params, take(enc, {1, 2, 3})); }));
        CHECK(throws_as<DuplicatePosition>([&] {
            decode_systematic(params, Codeword{{1, 5}, {1, 5}, {2, 6}, {3, 7}});
        }));
    }
    // systematic MDS over every k-subset, and the top field value (test_codec.cpp:192-224,333-339)
    {
        auto p = CodeParams::make(4, 8);
        auto src = random_source(4, 23);
        auto enc = encode_systematic(p, src);
        uint64_t ok = 0, pats = 0;
        for_each_subset(8, 4, [&](const std::vector<uint32_t>& keep) {
            ++pats;
            ok += decode_systematic(p, take(enc, keep)) == src;
        });
        CHECK(ok == pats && pats == 70);
        auto p3 = CodeParams::make(3, 7);
        std::vector<Fe> top{65536, 65536, 65536};
        auto enc3 = encode_systematic(p3, top);
        CHECK(decode_systematic(p3, take(enc3, {2, 4, 6})) == top);
    }
    // transform budgets at k = n/2, n = 4096 (acceptance.cpp:190-230, criterion 4)
    {
        const uint32_t k = 2048, n = 4096;
        auto sys = CodeParams::make(k, n, true), non = CodeParams::make(k, n, false);
        auto src = random_source(k, 404);
        auto enc_non = encode_nonsystematic(non, src);
        auto enc_sys = encode_systematic(sys, src);
        Codeword rx_non(k), rx_sys(k);
        for (uint32_t i = 0; i < k; ++i) {  // position 0 erased: no shortcuts
            rx_non[i] = {i + 1, enc_non[i + 1]};
            rx_sys[i] = {i + 1, enc_sys[i + 1]};
        }
        auto measure = [](auto&& op) {
            op();
            FntCounter counter;
            {
                FntScope scope(counter);
                op();
            }
            return counter.equivalents(4096);
        };
        const double e_non = measure([&] { encode_nonsystematic(non, src); });
        const double e_sys = measure([&] { encode_systematic(sys, src, Path::Fast); });
        const double d_non = measure([&] { CHECK(decode_nonsystematic(non, rx_non, Path::Fast) == src); });
        const double d_sys = measure([&] { CHECK(decode_systematic(sys, rx_sys, Path::Fast) == src); });
        std::printf("fnt budget: enc_nonsys=%.2f dec_nonsys=%.2f enc_sys=%.2f dec_sys=%.2f\n", e_non, d_non, e_sys,
                    d_sys);
        CHECK(e_non == 1.0 && d_non <= 8.0 && e_sys <= 9.0 && d_sys <= 9.0);
        // systematic prefix present: verbatim copy, zero transforms (test_codec.cpp:172-183)
        FntCounter counter;
        std::vector<Fe> got;
        {
            FntScope scope(counter);
            got = decode_systematic(sys, take(enc_sys, [&] {
                                        std::vector<uint32_t> p(k);
                                        for (uint32_t i = 0; i < k; ++i) p[i] = i;
                                        return p;
                                    }()));
        }
        CHECK(got == src && counter.total() == 0);
        // nested scopes both see a transform; a finished scope sees nothing more
        FntCounter outer, inner;
        {
            FntScope a(outer);
            {
                FntScope b(inner);
                encode_nonsystematic(non, src);
            }
            encode_nonsystematic(non, src);
        }
        CHECK(outer.count(4096) == 2 && inner.count(4096) == 1 && inner.total() == 1);
    }
    // transform API golden values (test_transform.cpp:28-71)
    {
        CHECK(fnt_forward(plan_for(2), std::vector<Fe>{1, 2}) == (std::vector<Fe>{3, 65536}));
        CHECK(fnt_forward(plan_for(4), std::vector<Fe>{9, 0, 0, 0}) == (std::vector<Fe>{9, 9, 9, 9}));
        CHECK(fnt_forward(plan_for(4), std::vector<Fe>{0, 1, 0, 0}) == (std::vector<Fe>{1, 65281, 65536, 256}));
        std::vector<Fe> x{1, 2, 3, 4, 5, 6, 7, 8};
        std::vector<Fe> want{36, 50109, 1020, 48061, 65533, 17468, 64509, 15420};
        CHECK(fnt_forward(plan_for(8), x) == want);
        CHECK(fnt_inverse(plan_for(8), want) == x);
        CHECK(throws_as<InvalidTransformSize>([] { plan_for(3); }));
        CHECK(throws_as<SizeMismatch>([] { fnt_forward(plan_for(8), std::vector<Fe>{1, 2}); }));
        // dif_forward / dit_inverse_unscaled compose into a cyclic convolution (transform.hpp:43-48)
        const uint32_t n = 64;
        auto a = random_source(n, 5), b = random_source(n, 6);
        std::vector<Fe> want_c(n, 0);
        for (uint32_t i = 0; i < n; ++i)
            for (uint32_t j = 0; j < n; ++j) want_c[(i + j) % n] = gf::add(want_c[(i + j) % n], gf::mul(a[i], b[j]));
        const auto& tp = plan_for(n);
        dif_forward(tp, a);
        dif_forward(tp, b);
        for (uint32_t i = 0; i < n; ++i) a[i] = gf::mul(gf::mul(a[i], b[i]), tp.size_inverse);
        dit_inverse_unscaled(tp, a);
        CHECK(a == want_c);
        CHECK(tp.root == gf::root_of_unity(n) && gf::mul(tp.root, tp.inverse_root) == 1);
    }
    // plan-level API golden values (test_interp.cpp:41-100)
    {
        using namespace fntrs::interp;
        std::vector<uint32_t> pos{0, 2, 5};
        DecodePlan plan = build_plan(8, pos);
        CHECK(plan.a() == (poly::Poly{16, 61169, 4351, 1}));
        CHECK(plan.aprime_at_x_inv == (std::vector<Fe>{gf::inv(4337), gf::inv(61712), gf::inv(3600)}));
        CHECK(plan.product_size == 8 && plan.a_fnt.size() == 8);
        CHECK(interpolate(plan, std::vector<Fe>{1000, 2000, 3000}) == (poly::Poly{46905, 62038, 23131}));
        CHECK(interpolate(build_plan(8, std::vector<uint32_t>{3}), std::vector<Fe>{321}) == poly::Poly{321});
        CHECK(interpolate(build_plan(4, std::vector<uint32_t>{0, 2}), std::vector<Fe>{12, 65535}) == (poly::Poly{5, 7}));
        auto cached = plan_for(8, std::vector<uint32_t>{5, 0, 2});
        CHECK(cached->positions == pos && plan_for(8, std::vector<uint32_t>{2, 5, 0}) == cached);
        CHECK(throws_as<TooFewPositions>([] { build_plan(8, std::vector<uint32_t>{}); }));
        CHECK(throws_as<PositionOutOfRange>([] { build_plan(8, std::vector<uint32_t>{1, 8}); }));
        CHECK(throws_as<DuplicatePosition>([] { build_plan(8, std::vector<uint32_t>{1, 1}); }));
        CHECK(throws_as<InvalidTransformSize>([] { build_plan(12, std::vector<uint32_t>{1}); }));
        CHECK(throws_as<SizeMismatch>([&] { interpolate(plan, std::vector<Fe>{1}); }));
    }
    // concurrent callers (test_transform.cpp:173-186): threads share the library
    // and get correct results; FntScope counts stay per thread
    {
        std::atomic<int> bad{0};
        std::vector<std::thread> pool;
        for (int t = 0; t < 4; ++t)
            pool.emplace_back([t, &bad] {
                const uint32_t k = 16u << t, n = 2 * k;
                auto p = CodeParams::make(k, n, t % 2 == 0);
                FntCounter counter;
                FntScope scope(counter);
                for (int r = 0; r < 10; ++r) {
                    auto src = random_source(k, 1000 * t + r);
                    auto enc = t % 2 == 0 ? encode_systematic(p, src) : encode_nonsystematic(p, src);
                    Codeword rx;
                    for (uint32_t i = r % 2; i < n; i += 2) rx.push_back({i, enc[i]});
                    auto dec = t % 2 == 0 ? decode_systematic(p, rx) : decode_nonsystematic(p, rx);
                    if (dec != src) ++bad;
                }
                // 10 encodes + 10 decodes on this thread only
                const uint64_t want = t % 2 == 0 ? 10 * 4 + 10 * 4 : 10 * 1 + 10 * 3;
                if (counter.total() != want) ++bad;
            });
        for (auto& th : pool) th.join();
        CHECK(bad.load() == 0);
    }
    // TransformPlan tables (transform.cpp:31-63) filled on the device
    {
        const auto& p8 = plan_for(8);
        CHECK(p8.twiddles == (std::vector<Fe>{1, 4096, 65281, 16}));  // r8 = 2^12, r8^3 = 2^36 = 16
        CHECK(p8.bit_reversal == (std::vector<uint32_t>{0, 4, 2, 6, 1, 5, 3, 7}));
        CHECK(p8.stage_twiddles == (std::vector<Fe>{1, 4096, 65281, 16, 1, 65281, 1}));
        for (uint32_t n : {1u, 2u, 1024u, 65536u}) {
            const auto& p = plan_for(n);
            bool ok = p.twiddles.size() == n / 2 && p.stage_twiddles.size() == (n > 1 ? n - 1 : 0);
            for (uint32_t j = 0; ok && j < n / 2; j += 97) ok = p.twiddles[j] == gf::pow(p.root, j) &&
                                                                  gf::mul(p.twiddles[j], p.inverse_twiddles[j]) == 1;
            size_t off = 0;
            for (uint32_t len = n; ok && len >= 2; len >>= 1) {
                for (uint32_t j = 0; j < len / 2; j += 31)
                    ok = ok && p.stage_twiddles[off + j] == p.twiddles[j * (n / len)] &&
                         p.stage_inverse_twiddles[off + j] == p.inverse_twiddles[j * (n / len)];
                off += len / 2;
            }
            CHECK(ok);
        }
    }
    // naive_dft (transform.cpp:325-343) against the fast transform; any root
    {
        std::mt19937_64 rng(11);
        for (uint32_t n : {1u, 8u, 256u, 1024u}) {
            std::vector<Fe> a(n);
            for (auto& x : a) x = Fe(rng() % 65537);
            CHECK(naive_dft(plan_for(n).root, a, false) == fnt_forward(plan_for(n), a));
            CHECK(naive_dft(plan_for(n).root, a, true) == fnt_inverse(plan_for(n), a));
        }
        CHECK(naive_dft(5, std::vector<Fe>{1, 1, 1}) == (std::vector<Fe>{3, 31, 651}));  // 1+5+25, 1+25+625
    }
    // subproduct tree / a() (test_interp.cpp:41-70 golden plan) and lagrange_oracle
    {
        auto plan = interp::build_plan(8, std::vector<uint32_t>{0, 2, 5});
        CHECK(plan.a() == (poly::Poly{16, 61169, 4351, 1}));
        CHECK(plan.a_tree.levels.size() == 3 && plan.a_tree.levels[0].size() == 3 &&
              plan.a_tree.levels[1].size() == 2 && plan.a_tree.levels[1][1] == plan.a_tree.levels[0][2]);
        std::mt19937_64 rng(12);
        for (uint32_t k : {1u, 7u, 64u, 300u}) {
            std::vector<std::pair<Fe, Fe>> pts;
            std::vector<uint32_t> pos;
            const uint32_t n = 1024;
            for (uint32_t z = 0; pos.size() < k; z += 1 + uint32_t(rng() % 3)) pos.push_back(z);
            std::vector<Fe> vals(k);
            for (uint32_t i = 0; i < k; ++i) {
                vals[i] = Fe(rng() % 65537);
                pts.push_back({gf::pow(plan_for(n).root, pos[i]), vals[i]});
            }
            auto pl = interp::build_plan(n, pos);
            CHECK(interp::interpolate(pl, vals) == interp::lagrange_oracle(pts));
            poly::Poly prod{1};
            for (auto& leaf : pl.a_tree.levels[0]) prod = poly::mul_schoolbook(prod, leaf);
            CHECK(prod == pl.a());
        }
        CHECK(throws_as<DuplicatePoint>([] { interp::lagrange_oracle(std::vector<std::pair<Fe, Fe>>{{3, 1}, {3, 2}}); }));
        CHECK(poly::derivative(poly::Poly{5, 3, 65536, 2}) == (poly::Poly{3, 65535, 6}));
        CHECK(poly::eval_horner(poly::Poly{1, 2, 3}, 10) == 321);
        CHECK(poly::middle_product(poly::Poly{1, 1}, poly::Poly{1, 2, 3}) == (std::vector<Fe>{3, 5}));
        CHECK(throws_as<ProductTooLarge>([] { poly::mul_fnt(poly::Poly(40000, 1), poly::Poly(40000, 1)); }));
    }
    // shard wire format golden bytes (test_shardio.cpp:70-87) and round trips
    {
        const shardio::ShardInfo info{7, 2, 4, 1, true};
        const auto b = shardio::write_shard(info, std::vector<Fe>{5, 65536, 7});
        const std::vector<uint8_t> want{'F', 'N', 'T', 'C', 1, 0, 0, 0, 0, 0, 0, 0, 7, 0, 2, 0, 4, 0, 1, 1,
                                        0, 0, 0, 3, 0, 1, 0, 0, 0, 1, 0, 5, 0, 0, 0, 7};
        CHECK(b == want);
        auto r = shardio::read_shard(b);
        CHECK(r.info == info && r.payload == (std::vector<Fe>{5, 65536, 7}));
        auto bad = b;
        bad[29] = 9;
        CHECK(throws_as<MalformedEscapes>([&] { shardio::read_shard(bad); }));
        const std::vector<uint8_t> data{1, 2, 3, 4, 5};
        auto m = shardio::symbolize(data, 2);
        CHECK(m.stripes == 2 && m.cells == (std::vector<Fe>{0x0102, 0x0304, 0x0500, 0}));
        CHECK(shardio::desymbolize(m, 5) == data);
        CHECK(throws_as<LengthMismatch>([&] { shardio::desymbolize(m, 9); }));
        const shardio::ChunkManifest man{9, 5, 2, 65536, 2, false};
        CHECK(shardio::read_manifest(shardio::write_manifest(man)) == man);
        CHECK(shardio::shard_filename(255, 3) == "00000000000000ff.3.fnt");
    }
    // geom.hpp: chirp evaluation (test_geom.cpp goldens and identities)
    {
        auto t4 = geom::build_chirp(4, gf::root_of_unity(4));
        CHECK(geom::geom_eval(std::vector<Fe>{9}, t4) == (std::vector<Fe>{9, 9, 9, 9}));
        CHECK(geom::geom_eval(std::vector<Fe>{5, 7}, geom::build_chirp(2, 65536)) == (std::vector<Fe>{12, 65535}));
        auto t1 = geom::build_chirp(1, 1);
        CHECK(geom::geom_eval(std::vector<Fe>{42}, t1) == (std::vector<Fe>{42}));
        CHECK(geom::geom_eval(std::vector<Fe>{}, t1) == (std::vector<Fe>{0}));
        auto t8 = geom::build_chirp(8, gf::root_of_unity(8));
        const std::vector<Fe> a{11, 22, 33, 44, 55, 66, 77, 88};
        CHECK(geom::geom_eval(a, t8) == (std::vector<Fe>{396, 26903, 11220, 4375, 65493, 61074, 54229, 38546}));
        CHECK(geom::geom_eval_negative(a, 8, gf::root_of_unity(8)) ==
              (std::vector<Fe>{38546, 54229, 61074, 65493, 4375, 11220, 26903, 396}));
        CHECK(geom::geom_eval_negative(std::vector<Fe>{0, 1}, 2, 65536) == (std::vector<Fe>{65536, 1}));
        CHECK(t8.b.size() == 15 && t8.b_inverse.size() == 8 && t8.b_fnt.size() == 16 && t8.b[0] == 1 && t8.b[1] == 1 &&
              t8.b[2] == gf::root_of_unity(8) && gf::mul(t8.b[5], t8.b_inverse[5]) == 1);
        CHECK(throws_as<SizeMismatch>([&] { geom::geom_eval(std::vector<Fe>(9, 1), t8); }));
        CHECK(throws_as<InvalidTransformSize>([] { geom::build_chirp(6, 3); }));
        std::mt19937_64 rng(31);
        for (uint32_t n = 1; n <= 256; n <<= 1) {  // any root, against Horner
            const Fe root = gf::root_of_unity(std::max(n, 4u));
            auto t = geom::build_chirp(n, root);
            std::vector<Fe> c(n);
            for (auto& x : c) x = Fe(rng() % 65537);
            auto got = geom::geom_eval(c, t);
            bool ok = true;
            for (uint32_t i = 0; i < n; ++i) ok = ok && got[i] == poly::eval_horner(c, gf::pow(root, i));
            CHECK(ok);
        }
        {
            std::vector<Fe> c(64);
            for (auto& x : c) x = Fe(rng() % 65537);
            CHECK(geom::geom_eval(c, geom::build_chirp(64, plan_for(64).root)) == fnt_forward(plan_for(64), c));
        }
        // cached table: two transforms per evaluation; the full domain: one
        auto t256 = geom::chirp_for(256, gf::root_of_unity(256));
        FntCounter c2;
        {
            FntScope scope(c2);
            geom::geom_eval(std::vector<Fe>(100, 3), *t256);
        }
        CHECK(c2.total() == 2 && c2.count(512) == 2);
        auto full = geom::chirp_for(65536, gf::root_of_unity(65536));
        CHECK(full->full_domain);
        std::vector<Fe> c(100);
        for (auto& x : c) x = Fe(rng() % 65537);
        FntCounter c1;
        std::vector<Fe> got;
        {
            FntScope scope(c1);
            got = geom::geom_eval(c, *full);
        }
        CHECK(c1.total() == 1 && c1.count(65536) == 1);
        const Fe r = gf::root_of_unity(65536), rinv = gf::inv(r);
        bool ok = true;
        for (uint32_t i : {0u, 1u, 2u, 100u, 65535u}) ok = ok && got[i] == poly::eval_horner(c, gf::pow(r, i));
        auto neg = geom::geom_eval_negative(c, 65536, r);
        for (uint32_t j : {0u, 1u, 7u, 65535u}) ok = ok && neg[j] == poly::eval_horner(c, gf::pow(rinv, j + 1));
        CHECK(ok);
    }
    std::printf("drop-in C++ API: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
