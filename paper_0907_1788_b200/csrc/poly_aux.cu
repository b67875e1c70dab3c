// poly_aux.cu -- the rest of the reference's public API on the GPU: the
// quadratic cross-checks (naive_dft, proj/src/transform.cpp:325-343;
// interp::lagrange_oracle, proj/src/interp.cpp:139-171), the TransformPlan
// tables (transform.cpp:31-63), the polynomial helpers behind poly.hpp
// (products, the subproduct tree, derivative, evaluation;
// proj/src/poly.cpp:22-242) and the element-wise steps of geom.hpp's chirp
// evaluation (proj/src/geom.cpp:13-116; its transforms are fntrs_gpu_fnt
// calls, capi.cu). None of these is on the batched codec path
// (the decoder replaces the tree by a log-domain convolution, DESIGN 4.4);
// they let the reference's own consumers (proj/tests/acceptance.cpp) link
// against the drop-in and get the reference's values, computed on the device.
//
// Arithmetic: canonical values in [0, p]; dot products accumulate exact
// uint64 sums of uint32 products (< 2^32 each, at most 2^16 terms -> < 2^48)
// and reduce once.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "field.cuh"
#include "fntrs_gpu.h"
#include "internal.h"

namespace fntrs_gpu {
namespace {

__device__ __forceinline__ uint32_t red64(uint64_t x) { return uint32_t(x % kP); }

// out[j] = sum_i a_i r^(ij) (r = root, or its inverse), then * (1/n) for the
// inverse; one thread per output, r^j by square-and-multiply, w stepped by r^j
// (the reference's loop order; any order gives the same field value)
__global__ void naive_dft_kernel(uint32_t r, uint32_t scale, uint32_t n, const uint32_t* __restrict__ in,
                                 uint32_t* __restrict__ out) {
    extern __shared__ uint32_t sa[];
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t rj = cpow(r, j);
    uint64_t acc = 0;
    uint32_t w = 1;
    for (uint32_t i0 = 0; i0 < n; i0 += 2048) {
        const uint32_t cnt = min(2048u, n - i0);
        __syncthreads();
        for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) sa[t] = in[i0 + t];
        __syncthreads();
        if (j < n)
            for (uint32_t t = 0; t < cnt; ++t) {
                acc += uint64_t(sa[t]) * w;
                w = cmul(w, rj);
                if ((t & 4095u) == 4095u) acc %= kP;
            }
        acc %= kP;
    }
    if (j < n) out[j] = cmul(red64(acc), scale);
}

// TransformPlan tables (transform.cpp:31-63): twiddles root^j and inverse
// twiddles for j < n/2, bit reversal, and the per-stage regrouping (the stage
// with block length len at offset n - len holds root^(j n/len), j < len/2)
__global__ void tables_kernel(uint32_t n, uint32_t bits, uint32_t root, uint32_t iroot, uint32_t* tw, uint32_t* itw,
                              uint32_t* bitrev, uint32_t* stw, uint32_t* sitw) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (i < n / 2) {
            if (tw) tw[i] = cpow(root, i);
            if (itw) itw[i] = cpow(iroot, i);
        }
        if (bitrev) bitrev[i] = bits ? __brev(i) >> (32 - bits) : 0u;
        if (i + 1 < n) {  // stage entry i: offset off(len) = n - len, j = i - off
            const uint32_t len = 1u << (32 - __clz(n - i - 1));  // next_pow2(n - i): n - len <= i < n - len/2
            const uint32_t j = i - (n - len), stride = n / len;
            if (stw) stw[i] = cpow(root, uint64_t(j) * stride);
            if (sitw) sitw[i] = cpow(iroot, uint64_t(j) * stride);
        }
    }
}

// Batched products of coefficient segments: block b computes outputs
// [chunk * 256, +256) of pair blk_pair[b]; out[j] = sum a_i b_{j-i}.
__global__ void pair_products_kernel(const fntrs_poly_pair* __restrict__ pairs, const uint32_t* __restrict__ blk_pair,
                                     const uint32_t* __restrict__ blk_chunk, const uint32_t* __restrict__ in,
                                     uint32_t* __restrict__ out) {
    const fntrs_poly_pair pr = pairs[blk_pair[blockIdx.x]];
    const uint32_t la = pr.a_len, lb = pr.b_len, lo = la + lb - 1;
    const uint32_t j = blk_chunk[blockIdx.x] * blockDim.x + threadIdx.x;
    if (!la || !lb || j >= lo) return;
    const uint32_t* a = in + pr.a_off;
    const uint32_t* b = in + pr.b_off;
    const uint32_t i0 = j >= lb ? j - lb + 1 : 0u, i1 = min(j, la - 1u);
    uint64_t acc = 0;
    for (uint32_t i = i0; i <= i1; ++i) acc += uint64_t(__ldg(a + i)) * __ldg(b + (j - i));
    out[pr.out_off + j] = red64(acc);
}

// (x - x_i) leaves: {p - x_i (mod p), 1}
__global__ void leaves_kernel(uint32_t k, const uint32_t* __restrict__ xs, uint32_t* __restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
        const uint32_t x = xs[i] % kP;
        out[2 * i] = x ? kP - x : 0u;
        out[2 * i + 1] = 1u;
    }
}

__global__ void copy_kernel(uint64_t n, const uint32_t* __restrict__ in, uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = in[i];
}

// Lagrange, per point i of a batch (thread per point): synthetic division of
// the master M (degree k, monic) by (x - x_i) from the top, evaluating the
// quotient at x_i by Horner in the same pass; scale_i = v_i / quotient(x_i).
// numer is stored [j][B] so a warp's writes are contiguous.
__global__ void lagrange_divide_kernel(uint32_t k, uint32_t i0, uint32_t B, const uint32_t* __restrict__ master,
                                       const uint32_t* __restrict__ xs, const uint32_t* __restrict__ vs,
                                       uint32_t* __restrict__ numer, uint32_t* __restrict__ scale) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= B || i0 + t >= k) return;
    const uint32_t xi = xs[i0 + t] % kP;
    uint32_t carry = master[k], h = 0;
    for (uint32_t j = k; j-- > 0;) {
        numer[size_t(j) * B + t] = carry;
        h = cmul(h, xi) + carry;
        h = h >= kP ? h - kP : h;
        const uint32_t c = cmul(xi, carry) + master[j];
        carry = c >= kP ? c - kP : c;
    }
    scale[t] = cmul(vs[i0 + t] % kP, cpow(h, kP - 2));
}

// out[j] += sum_t numer[j][t] scale[t]: one warp per j
__global__ void lagrange_accum_kernel(uint32_t k, uint32_t cnt, uint32_t B, const uint32_t* __restrict__ numer,
                                      const uint32_t* __restrict__ scale, uint32_t* __restrict__ out) {
    const uint32_t j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31u;
    if (j >= k) return;
    uint64_t acc = 0;
    for (uint32_t t = lane; t < cnt; t += 32) acc += uint64_t(numer[size_t(j) * B + t]) * scale[t];
    uint32_t r = red64(acc);
    for (int o = 16; o; o >>= 1) {
        r += __shfl_xor_sync(0xFFFFFFFFu, r, o);
        r = r >= kP ? r - kP : r;
    }
    if (lane == 0) {
        const uint32_t s = out[j] + r;
        out[j] = s >= kP ? s - kP : s;
    }
}

// formal derivative: out[i-1] = a_i * (i mod p)   (poly.cpp:201-208)
__global__ void derivative_kernel(uint32_t len, const uint32_t* __restrict__ a, uint32_t* __restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x + 1; i < len; i += gridDim.x * blockDim.x)
        out[i - 1] = cmul(a[i] % kP, i % kP);
}

// sum_i a_i x^i (poly.cpp:210-214 evaluates by Horner; same field value):
// one block, x^i by square-and-multiply per element, block reduction
__global__ void eval_kernel(uint32_t len, uint32_t x, const uint32_t* __restrict__ a, uint32_t* __restrict__ out) {
    __shared__ uint32_t part[32];
    uint64_t acc = 0;
    for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) acc += uint64_t(a[i] % kP) * cpow(x, i);
    uint32_t r = red64(acc);
    for (int o = 16; o; o >>= 1) {
        r += __shfl_xor_sync(0xFFFFFFFFu, r, o);
        r = r >= kP ? r - kP : r;
    }
    if ((threadIdx.x & 31u) == 0) part[threadIdx.x >> 5] = r;
    __syncthreads();
    if (threadIdx.x < 32) {
        r = threadIdx.x < blockDim.x / 32 ? part[threadIdx.x] : 0u;
        for (int o = 16; o; o >>= 1) {
            r += __shfl_xor_sync(0xFFFFFFFFu, r, o);
            r = r >= kP ? r - kP : r;
        }
        if (threadIdx.x == 0) *out = r;
    }
}

// ---- chirp (Bluestein) evaluation at geometric points (proj/src/geom.cpp) ----
// b_i = root^(i (i-1) / 2) (b_0 = 1, b_{i+1} = b_i root^i), b_inverse_i = 1 / b_i
__global__ void chirp_kernel(uint32_t n, uint32_t root, uint32_t* __restrict__ b, uint32_t* __restrict__ binv) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i + 1 < 2 * n; i += gridDim.x * blockDim.x) {
        const uint64_t e = uint64_t(i) * (i - (i ? 1u : 0u)) / 2;
        // root^65536 = 1 for root != 0 (Fermat); root = 0 gives b = 1, 1, 0, 0, ...
        const uint32_t v = root % kP ? cpow(root % kP, e % 65536u) : (i < 2 ? 1u : 0u);
        b[i] = v;
        if (i < n && binv) binv[i] = cpow(v, kP - 2);
    }
}

// c[n-1-j] = a_j / b_j for j < len, 0 elsewhere (2n entries)
__global__ void geom_pre_kernel(uint32_t n, uint32_t len, const uint32_t* __restrict__ a,
                                const uint32_t* __restrict__ binv, uint32_t* __restrict__ c) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < 2 * n; t += gridDim.x * blockDim.x) {
        uint32_t v = 0;
        if (t < n) {
            const uint32_t j = n - 1 - t;
            if (j < len) v = cmul(a[j] % kP, binv[j]);
        }
        c[t] = v;
    }
}

__global__ void pointwise_kernel(uint32_t m, uint32_t* __restrict__ c, const uint32_t* __restrict__ B) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x)
        c[t] = cmul(c[t], B[t]);
}

// out_i = c[n-1+i] / b_i
__global__ void geom_post_kernel(uint32_t n, const uint32_t* __restrict__ c, const uint32_t* __restrict__ binv,
                                 uint32_t* __restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = cmul(c[n - 1 + i], binv[i]);
}

// out_i = a_i rho^i (geom_eval_negative folds one power of rho into the coefficients)
__global__ void powers_scale_kernel(uint32_t len, uint32_t rho, const uint32_t* __restrict__ a,
                                    uint32_t* __restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x)
        out[i] = cmul(a[i] % kP, cpow(rho, i));
}

}  // namespace

unsigned grid_for(uint64_t n) { return unsigned(std::max<uint64_t>(1, std::min<uint64_t>(592, (n + 255) / 256))); }

cudaError_t launch_chirp(uint32_t n, uint32_t root, uint32_t* b, uint32_t* binv, cudaStream_t st) {
    chirp_kernel<<<grid_for(2ull * n), 256, 0, st>>>(n, root, b, binv);
    return cudaGetLastError();
}
cudaError_t launch_geom_pre(uint32_t n, uint32_t len, const uint32_t* a, const uint32_t* binv, uint32_t* c,
                            cudaStream_t st) {
    geom_pre_kernel<<<grid_for(2ull * n), 256, 0, st>>>(n, len, a, binv, c);
    return cudaGetLastError();
}
cudaError_t launch_pointwise(uint32_t m, uint32_t* c, const uint32_t* B, cudaStream_t st) {
    pointwise_kernel<<<grid_for(m), 256, 0, st>>>(m, c, B);
    return cudaGetLastError();
}
cudaError_t launch_geom_post(uint32_t n, const uint32_t* c, const uint32_t* binv, uint32_t* out, cudaStream_t st) {
    geom_post_kernel<<<grid_for(n), 256, 0, st>>>(n, c, binv, out);
    return cudaGetLastError();
}
cudaError_t launch_powers_scale(uint32_t len, uint32_t rho, const uint32_t* a, uint32_t* out, cudaStream_t st) {
    if (!len) return cudaSuccess;
    powers_scale_kernel<<<grid_for(len), 256, 0, st>>>(len, rho, a, out);
    return cudaGetLastError();
}

cudaError_t launch_naive_dft(uint32_t r, uint32_t scale, uint32_t n, const uint32_t* in, uint32_t* out,
                             cudaStream_t st) {
    if (!n) return cudaSuccess;
    naive_dft_kernel<<<(n + 255) / 256, 256, 2048 * 4, st>>>(r, scale, n, in, out);
    return cudaGetLastError();
}

cudaError_t launch_transform_tables(uint32_t n, uint32_t root, uint32_t iroot, uint32_t* tw, uint32_t* itw,
                                    uint32_t* bitrev, uint32_t* stw, uint32_t* sitw, cudaStream_t st) {
    uint32_t bits = 0;
    while ((1u << bits) < n) ++bits;
    tables_kernel<<<std::max(1u, std::min(592u, (n + 255) / 256)), 256, 0, st>>>(n, bits, root, iroot, tw, itw,
                                                                                    bitrev, stw, sitw);
    return cudaGetLastError();
}

// pairs: host array; in/out: device. Uploads the descriptors and the block map.
cudaError_t launch_pair_products(uint32_t npairs, const fntrs_poly_pair* pairs, const uint32_t* in, uint32_t* out,
                                 cudaStream_t st) {
    if (!npairs) return cudaSuccess;
    std::vector<uint32_t> bp, bc;
    for (uint32_t p = 0; p < npairs; ++p) {
        const uint64_t lo = (pairs[p].a_len && pairs[p].b_len) ? uint64_t(pairs[p].a_len) + pairs[p].b_len - 1 : 0;
        for (uint32_t c = 0; uint64_t(c) * 256 < lo; ++c) {
            bp.push_back(p);
            bc.push_back(c);
        }
    }
    if (bp.empty()) return cudaSuccess;
    const size_t nb = bp.size();
    char* buf = nullptr;
    const size_t bytes = npairs * sizeof(fntrs_poly_pair) + 2 * nb * 4 + 64;
    cudaError_t e = cudaMallocAsync(&buf, bytes, st);
    if (e) return e;
    auto* dpairs = reinterpret_cast<fntrs_poly_pair*>(buf);
    auto* dbp = reinterpret_cast<uint32_t*>(buf + npairs * sizeof(fntrs_poly_pair));
    auto* dbc = dbp + nb;
    e = cudaMemcpyAsync(dpairs, pairs, npairs * sizeof(fntrs_poly_pair), cudaMemcpyHostToDevice, st);
    if (!e) e = cudaMemcpyAsync(dbp, bp.data(), nb * 4, cudaMemcpyHostToDevice, st);
    if (!e) e = cudaMemcpyAsync(dbc, bc.data(), nb * 4, cudaMemcpyHostToDevice, st);
    // the host vectors die with this call: finish the uploads before returning
    if (!e) e = cudaStreamSynchronize(st);
    if (!e) {
        pair_products_kernel<<<unsigned(nb), 256, 0, st>>>(dpairs, dbp, dbc, in, out);
        e = cudaGetLastError();
    }
    cudaFreeAsync(buf, st);
    return e;
}

// Node lengths of the subproduct tree of k points, level by level
// (poly.cpp:216-242: pair adjacent nodes, carry an odd last node up).
std::vector<uint32_t> tree_node_lengths(uint32_t k, std::vector<uint32_t>* level_nodes) {
    std::vector<uint32_t> all, cur(k, 2u);
    if (level_nodes) level_nodes->clear();
    while (true) {
        all.insert(all.end(), cur.begin(), cur.end());
        if (level_nodes) level_nodes->push_back(uint32_t(cur.size()));
        if (cur.size() <= 1) break;
        std::vector<uint32_t> next;
        for (size_t i = 0; i + 1 < cur.size(); i += 2) next.push_back(cur[i] + cur[i + 1] - 1);
        if (cur.size() % 2) next.push_back(cur.back());
        cur.swap(next);
    }
    return all;
}

// All levels of the tree into `coeffs` (layout of tree_node_lengths).
cudaError_t launch_subproduct_tree(uint32_t k, const uint32_t* xs, uint32_t* coeffs, cudaStream_t st) {
    if (!k) return cudaSuccess;
    std::vector<uint32_t> lvl;
    const std::vector<uint32_t> len = tree_node_lengths(k, &lvl);
    leaves_kernel<<<std::max(1u, std::min(592u, (k + 255) / 256)), 256, 0, st>>>(k, xs, coeffs);
    cudaError_t e = cudaGetLastError();
    uint64_t node = 0, off = 0;  // first node / coefficient of the current level
    for (size_t l = 0; !e && l + 1 < lvl.size(); ++l) {
        const uint32_t cnt = lvl[l];
        uint64_t level_words = 0;
        for (uint32_t i = 0; i < cnt; ++i) level_words += len[node + i];
        std::vector<fntrs_poly_pair> pairs;
        uint64_t a = off, o = off + level_words;
        for (uint32_t i = 0; i + 1 < cnt; i += 2) {
            const uint32_t la = len[node + i], lb = len[node + i + 1];
            pairs.push_back({a, a + la, o, la, lb});
            a += la + lb;
            o += la + lb - 1;
        }
        e = launch_pair_products(uint32_t(pairs.size()), pairs.data(), coeffs, coeffs, st);
        if (!e && cnt % 2) {  // carried node
            const uint32_t lc = len[node + cnt - 1];
            copy_kernel<<<std::max(1u, std::min(592u, (lc + 255) / 256)), 256, 0, st>>>(lc, coeffs + a, coeffs + o);
            e = cudaGetLastError();
        }
        node += cnt;
        off += level_words;
    }
    return e;
}

cudaError_t launch_lagrange(uint32_t k, const uint32_t* xs, const uint32_t* vs, uint32_t* out, cudaStream_t st) {
    if (!k) return cudaSuccess;
    std::vector<uint32_t> lvl;
    const std::vector<uint32_t> len = tree_node_lengths(k, &lvl);
    uint64_t total = 0;
    for (uint32_t l : len) total += l;
    const uint32_t B = uint32_t(std::min<uint64_t>(k, std::max<uint64_t>(32, (uint64_t(1) << 26) / (k + 1))));
    uint32_t *tree = nullptr, *numer = nullptr;
    cudaError_t e = cudaMallocAsync(&tree, total * 4, st);
    if (!e) e = cudaMallocAsync(&numer, (size_t(k) * B + B) * 4, st);
    if (!e) e = launch_subproduct_tree(k, xs, tree, st);  // the master is the root, total - (k + 1)
    const uint32_t* master = tree + (total - (k + 1));
    if (!e) e = cudaMemsetAsync(out, 0, size_t(k) * 4, st);
    for (uint32_t i0 = 0; !e && i0 < k; i0 += B) {
        const uint32_t cnt = std::min(B, k - i0);
        uint32_t* scale = numer + size_t(k) * B;
        lagrange_divide_kernel<<<(cnt + 127) / 128, 128, 0, st>>>(k, i0, B, master, xs, vs, numer, scale);
        lagrange_accum_kernel<<<(k + 7) / 8, 256, 0, st>>>(k, cnt, B, numer, scale, out);
        e = cudaGetLastError();
    }
    if (numer) cudaFreeAsync(numer, st);
    if (tree) cudaFreeAsync(tree, st);
    return e;
}

cudaError_t launch_derivative(uint32_t len, const uint32_t* a, uint32_t* out, cudaStream_t st) {
    if (len <= 1) return cudaSuccess;
    derivative_kernel<<<std::max(1u, std::min(592u, (len + 255) / 256)), 256, 0, st>>>(len, a, out);
    return cudaGetLastError();
}

cudaError_t launch_eval(uint32_t len, uint32_t x, const uint32_t* a, uint32_t* out, cudaStream_t st) {
    eval_kernel<<<1, 1024, 0, st>>>(len, x % kP, a, out);
    return cudaGetLastError();
}

}  // namespace fntrs_gpu
