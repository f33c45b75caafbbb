// Broad phase (spatial hash + radix-sorted exact candidates), see geometry.cuh.
#include "geometry.cuh"

#include <cub/cub.cuh>

#include <cfloat>

#include "instrument.hpp"

namespace dabd_gpu {

namespace {

constexpr int kBlock = 128;

__global__ void k_inst_boxes(SceneView sc, InstView iv, int swept, double margin,
                             const double* dmargin, Box* box, double* cell_max) {
    if (dmargin) margin = *dmargin;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < iv.n; i += gridDim.x * blockDim.x) {
        const double mi = iv.skin ? margin + iv.skin[i] : margin;
        const int b = iv.body[i];
        const double* qa = iv.q0 + 6 * i;
        const double* qb = iv.q1 + 6 * i;
        Box bx{{DBL_MAX, DBL_MAX}, {-DBL_MAX, -DBL_MAX}};
        Box by = bx;
        for (int v = sc.vstart[b]; v < sc.vstart[b + 1]; ++v) {
            const V2 r = rest_of(sc, v);
            const V2 x = world_point(qa, r);
            bx.lo = vmin(bx.lo, x);
            bx.hi = vmax(bx.hi, x);
            if (swept) {
                const V2 y = world_point(qb, r);
                by.lo = vmin(by.lo, y);
                by.hi = vmax(by.hi, y);
            }
        }
        if (swept) bx = merge(bx, by);
        bx = inflate(bx, mi);
        box[i] = bx;
        if (!sc.is_static[b]) {
            const double ext = fmax(bx.hi.x - bx.lo.x, bx.hi.y - bx.lo.y);
            atomic_max_nonneg(cell_max, ext);
        }
    }
}

__device__ __forceinline__ unsigned cell_hash(int p, long long cx, long long cy, unsigned mask) {
    unsigned long long h = static_cast<unsigned long long>(cx) * 0x9E3779B97F4A7C15ull ^
                           static_cast<unsigned long long>(cy) * 0xC2B2AE3D27D4EB4Full ^
                           static_cast<unsigned long long>(p + 1) * 0x165667B19E3779F9ull;
    h ^= h >> 29;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 32;
    return static_cast<unsigned>(h) & mask;
}

__device__ __forceinline__ double inv_cell(const double* cell_max) {
    // 1.0001 slack keeps floor() cell indices within +-1 of each other for
    // overlapping boxes (rounding of x * inv).
    const double c = fmax(cell_max[0] * 1.0001, 1e-300);
    return 1.0 / c;
}

__global__ void k_hash_count(SceneView sc, InstView iv, const Box* box, const double* cell_max,
                             unsigned mask, int* hcount, int* hkey) {
    const double inv = inv_cell(cell_max);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < iv.n; i += gridDim.x * blockDim.x) {
        if (sc.is_static[iv.body[i]]) {
            hkey[i] = -1;
            continue;
        }
        const long long cx = static_cast<long long>(floor(box[i].lo.x * inv));
        const long long cy = static_cast<long long>(floor(box[i].lo.y * inv));
        const unsigned h = cell_hash(iv.part[i], cx, cy, mask);
        hkey[i] = static_cast<int>(h);
        atomicAdd(&hcount[h], 1);
    }
}

__global__ void k_hash_scatter(int n, const int* hkey, const int* hstart, int* hfill, int* items) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int h = hkey[i];
        if (h < 0) continue;
        items[hstart[h] + atomicAdd(&hfill[h], 1)] = i;
    }
}

// Candidates of the ordered pair (A -> B): points of A vs edges of B.
template <bool kWrite>
__device__ int emit_dir(const SceneView& sc, const InstView& iv, bool swept, double margin, int A,
                        int B, const KeyFmt& fmt, unsigned long long* out, int pos) {
    const int ba = iv.body[A], bb = iv.body[B];
    const double* qa0 = iv.q0 + 6 * A;
    const double* qa1 = iv.q1 + 6 * A;
    const double* qb0 = iv.q0 + 6 * B;
    const double* qb1 = iv.q1 + 6 * B;
    const int va0 = sc.vstart[ba], nva = sc.vstart[ba + 1] - va0;
    const int eb0 = sc.vstart[bb], neb = sc.vstart[bb + 1] - eb0;
    if (iv.skin) margin = (margin + iv.skin[A]) + iv.skin[B];
    int cnt = 0;
    for (int e = 0; e < neb; ++e) {
        const Box eb = edge_box(sc, qb0, qb1, swept, eb0 + e, margin);
        for (int v = 0; v < nva; ++v) {
            const Box pb = point_box(sc, qa0, qa1, swept, va0 + v);
            if (!overlaps(pb, eb)) continue;
            if (kWrite) out[pos + cnt] = fmt.pack(A, B, v, e);
            ++cnt;
        }
    }
    return cnt;
}

// Warp-cooperative emission: one warp per dynamic instance. Lanes 0..8 walk
// the 3x3 hash cells (and all lanes the statics) to collect overlapping
// partners; then the point x edge tests of each partner pair, both
// directions, are spread over the 32 lanes and compacted with ballots.
constexpr int kEmitWarps = 4;
constexpr int kMaxPartners = 96;

__device__ __forceinline__ bool combo_test(const SceneView& sc, const InstView& iv, bool swept,
                                           double margin, int A, int B, int c,
                                           const KeyFmt& fmt, unsigned long long& key) {
    const int ba = iv.body[A], bb = iv.body[B];
    const int va = sc.vstart[ba], na = sc.vstart[ba + 1] - va;
    const int vb = sc.vstart[bb], nbv = sc.vstart[bb + 1] - vb;
    int P = A, E = B, pv0 = va, ev0 = vb, ne = nbv;
    if (c >= na * nbv) { // second direction: points of B vs edges of A
        c -= na * nbv;
        P = B;
        E = A;
        pv0 = vb;
        ev0 = va;
        ne = na;
    }
    const int v = c / ne, e = c - v * ne;
    if (iv.skin) margin = (margin + iv.skin[P]) + iv.skin[E];
    const Box pb = point_box(sc, iv.q0 + 6 * P, iv.q1 + 6 * P, swept, pv0 + v);
    const Box eb = edge_box(sc, iv.q0 + 6 * E, iv.q1 + 6 * E, swept, ev0 + e, margin);
    if (!overlaps(pb, eb)) return false;
    key = fmt.pack(P, E, v, e);
    return true;
}

__global__ void __launch_bounds__(kEmitWarps * 32)
    k_emit_warp(SceneView sc, InstView iv, const Box* box, const double* cell_max, unsigned mask,
                const int* hstart, const int* hcount, const int* items, const int* stat,
                int n_stat, int swept, double margin, const double* dmargin, KeyFmt fmt,
                unsigned long long* out, int cap, int* counter, int* err) {
    if (dmargin) margin = *dmargin;
    __shared__ int partners[kEmitWarps][kMaxPartners];
    __shared__ int npart[kEmitWarps];
    __shared__ int wtot[kEmitWarps];
    __shared__ int base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool sw = swept != 0;
    const double inv = inv_cell(cell_max);
    for (int start = blockIdx.x * kEmitWarps; start < iv.n; start += gridDim.x * kEmitWarps) {
        const int i = start + warp;
        if (lane == 0) npart[warp] = 0;
        __syncwarp();
        const bool valid = i < iv.n && !sc.is_static[iv.body[i]];
        if (valid) {
            const Box bi = box[i];
            const int p = iv.part[i];
            const long long cx0 = static_cast<long long>(floor(bi.lo.x * inv)) - 1;
            const long long cy0 = static_cast<long long>(floor(bi.lo.y * inv)) - 1;
            const long long cx1 = static_cast<long long>(floor(bi.hi.x * inv));
            const long long cy1 = static_cast<long long>(floor(bi.hi.y * inv));
            const long long cx = cx0 + lane / 3, cy = cy0 + lane % 3;
            const bool cell_ok = lane < 9 && cx <= cx1 && cy <= cy1;
            const unsigned h = cell_ok ? cell_hash(p, cx, cy, mask) : 0xffffffffu;
            bool dup = false;
#pragma unroll
            for (int m = 0; m < 9; ++m) {
                const unsigned hm = __shfl_sync(0xffffffffu, h, m);
                if (m < lane && cell_ok && hm == h) dup = true;
            }
            if (cell_ok && !dup) {
                const int s0 = hstart[h], s1 = s0 + hcount[h];
                for (int t = s0; t < s1; ++t) {
                    const int j = items[t];
                    if (j <= i || iv.part[j] != p || !overlaps(bi, box[j])) continue;
                    const int slot = atomicAdd(&npart[warp], 1);
                    if (slot < kMaxPartners) partners[warp][slot] = j;
                }
            }
            for (int k = lane; k < n_stat; k += 32) {
                const int s = stat[k];
                if (iv.part[s] != p || !overlaps(bi, box[s])) continue;
                const int slot = atomicAdd(&npart[warp], 1);
                if (slot < kMaxPartners) partners[warp][slot] = s;
            }
        }
        __syncwarp();
        const int np_raw = npart[warp];
        // Partners of instance i: the shared-memory list, or (more than
        // kMaxPartners, e.g. a large body resting on many small ones) the
        // same hash cells and statics walked again warp-uniformly. Either way
        // every partner is visited once; the keys are sorted afterwards, so
        // the visiting order does not matter.
        const bool spill = np_raw > kMaxPartners;
        const int np = min(np_raw, kMaxPartners);
        auto for_each_partner = [&](auto&& fn) {
            if (!valid) return;
            if (!spill) {
                for (int q = 0; q < np; ++q) fn(partners[warp][q]);
                return;
            }
            const Box bi = box[i];
            const int p = iv.part[i];
            const long long cx0 = static_cast<long long>(floor(bi.lo.x * inv)) - 1;
            const long long cy0 = static_cast<long long>(floor(bi.lo.y * inv)) - 1;
            const long long cx1 = static_cast<long long>(floor(bi.hi.x * inv));
            const long long cy1 = static_cast<long long>(floor(bi.hi.y * inv));
            unsigned seen[9];
            int nseen = 0;
            for (int m = 0; m < 9; ++m) {
                const long long cx = cx0 + m / 3, cy = cy0 + m % 3;
                if (cx > cx1 || cy > cy1) continue;
                const unsigned h = cell_hash(p, cx, cy, mask);
                bool dup = false;
                for (int u = 0; u < nseen; ++u) dup = dup || seen[u] == h;
                if (dup) continue;
                seen[nseen++] = h;
                const int s0 = hstart[h], s1 = s0 + hcount[h];
                for (int t = s0; t < s1; ++t) {
                    const int j = items[t];
                    if (j <= i || iv.part[j] != p || !overlaps(bi, box[j])) continue;
                    fn(j);
                }
            }
            for (int k = 0; k < n_stat; ++k) {
                const int st = stat[k];
                if (iv.part[st] != p || !overlaps(bi, box[st])) continue;
                fn(st);
            }
        };
        // count pass
        int cnt = 0;
        for_each_partner([&](int j) {
            const int na = sc.vstart[iv.body[i] + 1] - sc.vstart[iv.body[i]];
            const int nb = sc.vstart[iv.body[j] + 1] - sc.vstart[iv.body[j]];
            const int combos = 2 * na * nb;
            for (int c = lane; c < combos; c += 32) {
                unsigned long long k;
                cnt += combo_test(sc, iv, sw, margin, i, j, c, fmt, k) ? 1 : 0;
            }
        });
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
        if (lane == 0) wtot[warp] = cnt;
        __syncthreads();
        if (threadIdx.x == 0) {
            int total = 0;
            for (int w = 0; w < kEmitWarps; ++w) total += wtot[w];
            base = atomicAdd(&counter[0], total);
            if (base + total > cap) {
                atomicMax(&counter[1], base + total);
                if (err) raise(err, kErrCapacity);
                base = -1;
            }
        }
        __syncthreads();
        if (base >= 0) {
            int pos = base;
            for (int w = 0; w < warp; ++w) pos += wtot[w];
            for_each_partner([&](int j) {
                const int na = sc.vstart[iv.body[i] + 1] - sc.vstart[iv.body[i]];
                const int nb = sc.vstart[iv.body[j] + 1] - sc.vstart[iv.body[j]];
                const int combos = 2 * na * nb;
                for (int cb = 0; cb < combos; cb += 32) {
                    const int c = cb + lane;
                    unsigned long long k = 0;
                    const bool hit = c < combos && combo_test(sc, iv, sw, margin, i, j, c, fmt, k);
                    const unsigned bal = __ballot_sync(0xffffffffu, hit);
                    if (hit) out[pos + __popc(bal & ((1u << lane) - 1u))] = k;
                    pos += __popc(bal);
                }
            });
        }
        __syncthreads();
    }
}

__global__ void k_emit_static_pairs(SceneView sc, InstView iv, const Box* box, const int* stat,
                                    int n_stat, int swept, double margin, const double* dmargin,
                                    KeyFmt fmt, unsigned long long* out, int cap, int* counter,
                                    int* err) {
    if (dmargin) margin = *dmargin;
    const long long np = static_cast<long long>(n_stat) * n_stat;
    for (long long t = blockIdx.x * blockDim.x + threadIdx.x; t < np;
         t += gridDim.x * blockDim.x) {
        const int i = stat[t / n_stat], j = stat[t % n_stat];
        if (j <= i || iv.part[i] != iv.part[j] || !overlaps(box[i], box[j])) continue;
        const int c = emit_dir<false>(sc, iv, swept != 0, margin, i, j, fmt, nullptr, 0) +
                      emit_dir<false>(sc, iv, swept != 0, margin, j, i, fmt, nullptr, 0);
        const int pos = atomicAdd(&counter[0], c);
        if (pos + c > cap) {
            atomicMax(&counter[1], pos + c);
            if (err) raise(err, kErrCapacity);
            continue;
        }
        const int c1 = emit_dir<true>(sc, iv, swept != 0, margin, i, j, fmt, out, pos);
        emit_dir<true>(sc, iv, swept != 0, margin, j, i, fmt, out, pos + c1);
    }
}

// On overflow the blocks that did not fit left their reserved slots at the
// 0xFF padding, whose keys decode to instance ids past the table: the list
// is emptied (counter[1] keeps the size needed) so no consumer decodes them
// before the host sees kErrCapacity and redoes the work with a larger list.
__global__ void k_list_overflow_guard(int* counter, int cap) {
    if (threadIdx.x == 0 && counter[0] > cap) {
        atomicMax(&counter[1], counter[0]);
        counter[0] = 0;
    }
}

// narrow_phase over an explicit body-level candidate list (geometry.cpp:210-228).
__global__ void k_narrow_bodies(SceneView sc, const double* q, const int* cand, int n,
                                double d_hat, double* d, int* flag, int* err) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const int a = cand[4 * t], b = cand[4 * t + 1], v = cand[4 * t + 2], e = cand[4 * t + 3];
        const int vf = sc.vstart[a] + v, ef = sc.vstart[b] + e;
        const V2 P = world_point(q + 6 * a, rest_of(sc, vf));
        const V2 E0 = world_point(q + 6 * b, rest_of(sc, ef));
        const V2 E1 = world_point(q + 6 * b, rest_of(sc, sc.vnext[ef]));
        const double dd = pe_distance(P, E0, E1);
        if (dd == -1.0) raise(err, kErrDegenerateEdge);
        d[t] = dd;
        flag[t] = dd < d_hat ? 1 : 0;
    }
}

} // namespace

void launch_narrow_bodies(const SceneView& sc, const double* q, const int* cand, int n,
                          double d_hat, double* d, int* flag, int* err, cudaStream_t s) {
    if (n == 0) return;
    DABD_LAUNCH("k_narrow_bodies", s, k_narrow_bodies<<<grid_for(n, kBlock), kBlock, 0, s>>>(sc, q, cand, n, d_hat, d, flag, err));
}

void launch_inst_boxes(const SceneView& sc, const InstView& iv, bool swept, double margin, Box* box,
                       double* cell_max, cudaStream_t s, const double* dmargin) {
    if (iv.n == 0) return;
    DABD_LAUNCH("k_inst_boxes", s, k_inst_boxes<<<grid_for(iv.n, kBlock), kBlock, 0, s>>>(sc, iv, swept ? 1 : 0, margin,
                                                          dmargin, box, cell_max));
}

Detector::Detector() {
    cell_.resize(1);
    counter_.resize(2);
    pin_.resize(4);
}

Detector::~Detector() = default;

void Detector::prepare(int n_inst, int max_verts, int cap) {
    fmt_.ibits = bits_for(std::max(n_inst, 2));
    fmt_.vbits = bits_for(std::max(max_verts, 2));
    if (fmt_.total_bits() > 64) throw Error("broad phase: instance/vertex counts exceed key width");
    unsigned tsize = 1;
    while (tsize < 2u * static_cast<unsigned>(std::max(n_inst, 1))) tsize <<= 1;
    tsize_ = tsize;
    cap = std::max(cap, 64);
    box_.resize(std::max(n_inst, 1));
    n_cap_ = std::max(n_inst, 1);
    hcount_.resize(tsize);
    hstart_.resize(tsize);
    hfill_.resize(tsize);
    hitems_.resize(std::max(n_inst, 1));
    hkey_.resize(std::max(n_inst, 1));
    keys_.resize(cap);
    keys_sorted_.resize(cap);
    cap_ = cap;
    size_t tb = 0, sb = 0;
    CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tb, hcount_.get(), hstart_.get(),
                                             static_cast<int>(tsize)));
    CUDA_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, sb, keys_.get(), keys_sorted_.get(), cap, 0,
                                              fmt_.total_bits()));
    temp_.resize(std::max(tb, sb));
    temp_bytes_ = std::max(tb, sb);
}

void Detector::enqueue(const SceneView& sc, const InstView& iv, const int* stat, int n_stat,
                       bool swept, double margin, int* err, cudaStream_t s, const double* dmargin) {
    CUDA_CHECK(cudaMemsetAsync(counter_.get(), 0, 2 * sizeof(int), s));
    CUDA_CHECK(cudaMemsetAsync(keys_sorted_.get(), 0xFF, sizeof(unsigned long long) * cap_, s));
    if (iv.n == 0) return;
    CUDA_CHECK(cudaMemsetAsync(cell_.get(), 0, sizeof(double), s));
    launch_inst_boxes(sc, iv, swept, margin, box_.get(), cell_.get(), s, dmargin);
    CUDA_CHECK(cudaMemsetAsync(hcount_.get(), 0, sizeof(int) * tsize_, s));
    DABD_LAUNCH("k_hash_count", s,
                k_hash_count<<<grid_for(iv.n, kBlock), kBlock, 0, s>>>(
                    sc, iv, box_.get(), cell_.get(), tsize_ - 1, hcount_.get(), hkey_.get()));
    size_t tb = temp_bytes_;
    CUDA_CHECK(cub::DeviceScan::ExclusiveSum(temp_.get(), tb, hcount_.get(), hstart_.get(),
                                             static_cast<int>(tsize_), s));
    CUDA_CHECK(cudaMemsetAsync(hfill_.get(), 0, sizeof(int) * tsize_, s));
    DABD_LAUNCH("k_hash_scatter", s,
                k_hash_scatter<<<grid_for(iv.n, kBlock), kBlock, 0, s>>>(
                    iv.n, hkey_.get(), hstart_.get(), hfill_.get(), hitems_.get()));
    CUDA_CHECK(cudaMemsetAsync(keys_.get(), 0xFF, sizeof(unsigned long long) * cap_, s));
    DABD_LAUNCH("k_emit", s,
                k_emit_warp<<<grid_for(iv.n, kEmitWarps, 148 * 64), kEmitWarps * 32, 0, s>>>(
                    sc, iv, box_.get(), cell_.get(), tsize_ - 1, hstart_.get(), hcount_.get(),
                    hitems_.get(), stat, n_stat, swept ? 1 : 0, margin, dmargin, fmt_, keys_.get(), cap_,
                    counter_.get(), err));
    if (n_stat > 1) {
        const int gs = grid_for(static_cast<long long>(n_stat) * n_stat, kBlock);
        DABD_LAUNCH("k_emit_static_pairs", s,
                    k_emit_static_pairs<<<gs, kBlock, 0, s>>>(sc, iv, box_.get(), stat, n_stat,
                                                              swept ? 1 : 0, margin, dmargin, fmt_,
                                                              keys_.get(), cap_, counter_.get(),
                                                              err));
    }
    DABD_LAUNCH("k_list_overflow_guard", s, k_list_overflow_guard<<<1, 32, 0, s>>>(counter_.get(), cap_));
    size_t sb = temp_bytes_;
    CUDA_CHECK(cub::DeviceRadixSort::SortKeys(temp_.get(), sb, keys_.get(), keys_sorted_.get(), cap_,
                                              0, fmt_.total_bits(), s));
}

void Detector::ensure(int n_inst, int max_verts, int cap) {
    // per-instance buffers too: a set that grew within the hash table's slack
    // would otherwise write boxes / hash items past their allocation
    if (cap != cap_ || n_inst > n_cap_ || tsize_ < 2u * static_cast<unsigned>(std::max(n_inst, 1)) ||
        fmt_.ibits != bits_for(std::max(n_inst, 2)) || fmt_.vbits != bits_for(std::max(max_verts, 2)))
        prepare(n_inst, max_verts, cap);
}

int Detector::build(const SceneView& sc, const InstView& iv, const int* stat, int n_stat,
                    bool swept, double margin, int max_verts, cudaStream_t s) {
    int cap = std::max(cap_, 64 * std::max(iv.n, 1));
    for (int attempt = 0; attempt < 4; ++attempt) {
        if (cap != cap_ || iv.n > n_cap_ || tsize_ < 2u * static_cast<unsigned>(std::max(iv.n, 1)) ||
            fmt_.ibits != bits_for(std::max(iv.n, 2)) || fmt_.vbits != bits_for(std::max(max_verts, 2)))
            prepare(iv.n, max_verts, cap);
        enqueue(sc, iv, stat, n_stat, swept, margin, nullptr, s);
        CUDA_CHECK(cudaMemcpyAsync(pin_.get(), counter_.get(), 2 * sizeof(int),
                                   cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        if (pin_[1] == 0 && pin_[0] <= cap_) { // (the guard empties an overflowed list)
            count_ = pin_[0];
            return count_;
        }
        cap = std::max(pin_[0], pin_[1]) + cap_ / 4;
    }
    throw Error("broad phase: candidate buffer growth failed");
}

} // namespace dabd_gpu
