// Slab partitions, requirement masks and span layouts on the GPU
// (proj/src/partitioner.cpp:46-218), bit-exact with the reference.
#include "gmd_partition.cuh"

#include <vector>

namespace gmd {
namespace {

// ---------------------------------------------------------------------------
// Quantile radix select (partitioner.cpp:77-85 needs only the order
// statistics s[c-1], s[c] of the sorted wrapped fractions, never the full
// sort).  Keys are non-negative doubles, so their bit patterns order as u64.
// ---------------------------------------------------------------------------
constexpr int kSelMaxRanks = 2 * kMaxParts;
constexpr int kSelSmemGroups = 40;

struct SelState {
    unsigned long long prefix[kSelMaxRanks];
    long long rem[kSelMaxRanks];
    unsigned long long ugroup[kSelMaxRanks];
    int gmap[kSelMaxRanks];
    int ng;
    int nr;
};

__device__ __forceinline__ int find_group(const SelState& st, unsigned long long kp) {
    int lo = 0, hi = st.ng - 1;
    while (lo <= hi) {
        int mid = (lo + hi) >> 1;
        unsigned long long v = st.ugroup[mid];
        if (v == kp) return mid;
        if (v < kp) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

// One radix pass as one launch: every CTA histograms its keys (shared-memory
// privatized), and the last CTA to finish (atomic ticket) performs the
// update -- per rank, a warp prefix-scans the 256 digit counts to find the
// digit holding the rank -- then clears the histogram and regroups the
// ranks by prefix.  One launch per pass
// and no serial 256-step scan per pass (the two-launch form cost 0.24 ms
// per build at C5, 8 x (hist 10 us + update 19 us)).
__global__ void k_sel_pass(const unsigned long long* __restrict__ keys, int64_t n, SelState* stp,
                           unsigned int* hist, unsigned int* ticket, int shift, double* out, int last) {
    __shared__ SelState st;
    __shared__ unsigned int sh[kSelSmemGroups * 256];
    __shared__ bool am_last;
    for (int k = threadIdx.x; k < (int)(sizeof(SelState) / 4); k += blockDim.x)
        reinterpret_cast<int*>(&st)[k] = reinterpret_cast<const int*>(stp)[k];
    __syncthreads();
    const bool use_sm = st.ng <= kSelSmemGroups;
    if (use_sm)
        for (int k = threadIdx.x; k < st.ng * 256; k += blockDim.x) sh[k] = 0;
    __syncthreads();
    const unsigned long long mask_hi = shift >= 56 ? 0ull : ~((1ull << (shift + 8)) - 1ull);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = keys[i];
        const int g = find_group(st, key & mask_hi);
        if (g < 0) continue;
        const int slot = g * 256 + (int)((key >> shift) & 255ull);
        if (use_sm)
            atomicAdd(&sh[slot], 1u);
        else
            atomicAdd(&hist[slot], 1u);
    }
    if (use_sm) {
        __syncthreads();
        for (int k = threadIdx.x; k < st.ng * 256; k += blockDim.x)
            if (sh[k]) atomicAdd(&hist[k], sh[k]);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) am_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    for (int k = warp; k < st.nr; k += nwarp) {
        const unsigned int* h = hist + st.gmap[k] * 256;
        unsigned int c[8];
        long long mine = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            c[i] = __ldcg(h + 8 * lane + i);
            mine += c[i];
        }
        long long incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        const long long rem = st.rem[k], excl = incl - mine;
        const long long total = __shfl_sync(0xffffffffu, incl, 31);
        // first digit d with cum(d) + h[d] > rem (else 255, cum = total)
        const unsigned owner = __ballot_sync(0xffffffffu, excl <= rem && rem < incl);
        if (owner == 0u) {
            if (lane == 0) {
                stp->prefix[k] = st.prefix[k] | (255ull << shift);
                stp->rem[k] = rem - total;
            }
        } else if (lane == __ffs(owner) - 1) {
            long long cum = excl;
            int digit = 8 * lane + 7;
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (cum + (long long)c[i] > rem) {
                    digit = 8 * lane + i;
                    break;
                } else {
                    cum += c[i];
                }
            stp->prefix[k] = st.prefix[k] | ((unsigned long long)digit << shift);
            stp->rem[k] = rem - cum;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < st.ng * 256; i += blockDim.x) hist[i] = 0;
    if (threadIdx.x == 0) {
        *ticket = 0u;
        int ng = 0;
        for (int r = 0; r < st.nr; ++r) {
            const unsigned long long pr = stp->prefix[r];
            if (ng == 0 || stp->ugroup[ng - 1] != pr) stp->ugroup[ng++] = pr;
            stp->gmap[r] = ng - 1;
            if (last) out[r] = __longlong_as_double((long long)pr);
        }
        stp->ng = ng;
    }
}

// ---------------------------------------------------------------------------
// owners, requirement masks
// ---------------------------------------------------------------------------
__global__ void k_owner(const double* __restrict__ fw, int64_t n, const Bounds bd,
                        int32_t* __restrict__ owner) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double f = fw[i];
    int o;
    if (f >= 1.0) {
        o = bd.p - 1;
    } else {  // upper_bound over b[1..p-1] (partitioner.cpp:93-100)
        int lo = 1, hi = bd.p;  // first k in [1, p) with b[k] > f, else p
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (bd.b[mid] > f) hi = mid; else lo = mid + 1;
        }
        o = lo - 1;
    }
    owner[i] = o;
}

__global__ void k_required(const int32_t* __restrict__ row, const int32_t* __restrict__ src,
                           int64_t n, const int32_t* __restrict__ owner,
                           unsigned long long* __restrict__ req) {
    int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (v >= n) return;
    const int ov = owner[v];
    for (int e = row[v] + (threadIdx.x & 31); e < row[v + 1]; e += 32) {
        int u = src[e];
        if (owner[u] != ov) atomicOr(&req[u], 1ull << ov);
    }
}

// One rank per GPU: only the rank's own rows exist.  FROM bits come straight
// from the rows (an in-edge u -> v of an owned v marks u as required by r,
// partitioner.cpp:124-134); TO bits of an owned v use the reverse edge (every
// edge u -> v has the reverse v -> u, neighborlist symmetry).
__global__ void k_required_rank(const int32_t* __restrict__ row, const int32_t* __restrict__ src,
                                int64_t n, const int32_t* __restrict__ owner, int r,
                                unsigned long long* __restrict__ req) {
    int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (v >= n || owner[v] != r) return;
    unsigned long long m = 0ull;
    for (int e = row[v] + (threadIdx.x & 31); e < row[v + 1]; e += 32) {
        const int u = src[e];
        const int ou = owner[u];
        if (ou != r) {
            atomicOr(&req[u], 1ull << r);
            m |= 1ull << ou;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m |= __shfl_xor_sync(0xffffffffu, m, o);
    if ((threadIdx.x & 31) == 0 && m) atomicOr(&req[v], m);
}

__global__ void k_flag_owned(const int32_t* __restrict__ owner, int64_t n, int r,
                             int32_t* __restrict__ flag) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) flag[v] = owner[v] == r ? 1 : 0;
}

__global__ void k_compact_owned(const int32_t* __restrict__ owner, int64_t n, int r,
                                const int32_t* __restrict__ pos, int32_t* __restrict__ nodes) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n && owner[v] == r) nodes[pos[v]] = (int32_t)v;
}

// interior atoms of rank r: every in-edge source owned by r, so their
// layer update reads no halo row and can run while the halo is in flight
__global__ void k_flag_interior(int64_t n_own, const int32_t* __restrict__ nodes,
                                const int32_t* __restrict__ row, const int32_t* __restrict__ src,
                                const int32_t* __restrict__ owner, int r, int32_t* __restrict__ flag) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_own) return;
    const int v = nodes[k];
    int in = 1;
    for (int e = row[v]; e < row[v + 1] && in; ++e) in = owner[src[e]] == r;
    flag[k] = in;
}

// stable split: interior atoms first, then the border atoms, ascending in each
__global__ void k_split_nodes(int64_t n_own, const int32_t* __restrict__ nodes,
                              const int32_t* __restrict__ pos, int32_t* __restrict__ out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_own) return;
    const int64_t n_int = pos[n_own];
    out[pos[k + 1] > pos[k] ? pos[k] : n_int + k - pos[k]] = nodes[k];
}

// send plan: canonical row of every TO row of partition r (TO region rows
// [t0, t1) of the super layout)
__global__ void k_send_rows(int32_t t0, int32_t t1, const int32_t* __restrict__ node_array,
                            const int32_t* __restrict__ crow, int32_t* __restrict__ xsend) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (t0 + k < t1) xsend[k] = crow[node_array[t0 + k]];
}

// ---------------------------------------------------------------------------
// stable multi-list compaction (build_span_layout, partitioner.cpp:153-180)
// ---------------------------------------------------------------------------
constexpr int kChunk = 256;  // ids per warp-chunk (C5 p = 8: 3888 warps, ~26 per SM; 1024: 972)

// smallest list id > last that node (owner o, mask m) belongs to, or INT_MAX
__device__ __forceinline__ int next_list(int o, unsigned long long m, int p, int last) {
    const int stride = 1 + 2 * p;
    int best = 0x7fffffff;
    if (m == 0ull) {
        int l = o * stride;
        if (l > last) best = l;
    } else {
        int t = last - o * stride - 1;  // need j > t
        unsigned long long mm = t < 0 ? m : (t >= 63 ? 0ull : (m & (~0ull << (t + 1))));
        if (mm) best = o * stride + 1 + __ffsll((long long)mm) - 1;
    }
    if (m != 0ull) {
        int a = last - 1 - p - o;  // need i*stride > a
        int t2 = a >= 0 ? a / stride : -((-a + stride - 1) / stride);
        unsigned long long mm = t2 < 0 ? m : (t2 >= 63 ? 0ull : (m & (~0ull << (t2 + 1))));
        if (mm) {
            int l = (__ffsll((long long)mm) - 1) * stride + 1 + p + o;
            if (l < best) best = l;
        }
    }
    return best;
}

// memberships restricted to partition `only` (>= 0), i.e. lists
// [only*stride, (only+1)*stride); only < 0 keeps every partition
__device__ __forceinline__ int next_list_only(int o, unsigned long long m, int p, int last,
                                              int only) {
    const int stride = 1 + 2 * p;
    int l = next_list(o, m, p, last);
    if (only >= 0)
        while (l != 0x7fffffff && l / stride != only) l = next_list(o, m, p, l);
    return l;
}

__global__ void k_lay_count(const int32_t* __restrict__ owner,
                            const unsigned long long* __restrict__ req, int64_t nid, int p,
                            int nlists, int64_t nchunks, int32_t* __restrict__ counts, int only) {
    extern __shared__ int cnt[];
    for (int l = threadIdx.x; l < nlists; l += 32) cnt[l] = 0;
    __syncwarp();
    const int64_t c = blockIdx.x;
    const int64_t b0 = c * kChunk, b1 = min(nid, b0 + kChunk);
    for (int64_t v = b0 + threadIdx.x; v < b1; v += 32) {
        int o = owner[v];
        unsigned long long m = req[v];
        for (int l = next_list_only(o, m, p, -1, only); l != 0x7fffffff;
             l = next_list_only(o, m, p, l, only))
            atomicAdd(&cnt[l], 1);
    }
    __syncwarp();
    for (int l = threadIdx.x; l < nlists; l += 32) counts[(int64_t)l * nchunks + c] = cnt[l];
}

__global__ void k_lay_scatter(const int32_t* __restrict__ owner,
                              const unsigned long long* __restrict__ req, int64_t nid, int p,
                              int nlists, int64_t nchunks, const int32_t* __restrict__ offs,
                              int32_t* __restrict__ node_array, int32_t* __restrict__ crow,
                              int only) {
    extern __shared__ int run[];
    const int lane = threadIdx.x;
    for (int l = lane; l < nlists; l += 32) run[l] = 0;
    __syncwarp();
    const int64_t c = blockIdx.x;
    const int64_t b0 = c * kChunk, b1 = min(nid, b0 + kChunk);
    const int stride = 1 + 2 * p;
    for (int64_t vb = b0; vb < b1; vb += 32) {
        const int64_t v = vb + lane;
        const bool valid = v < b1;
        int o = valid ? owner[v] : 0;
        unsigned long long m = valid ? req[v] : 0ull;
        int cur = valid ? next_list_only(o, m, p, -1, only) : 0x7fffffff;
        const int canon = m == 0ull ? o * stride : o * stride + __ffsll((long long)m);
        while (true) {
            int lmin = (int)__reduce_min_sync(0xffffffffu, (unsigned)cur);
            if (lmin == 0x7fffffff) break;
            bool mine = cur == lmin;
            unsigned bal = __ballot_sync(0xffffffffu, mine);
            if (mine) {
                int rank = __popc(bal & ((1u << lane) - 1u));
                int pos = offs[(int64_t)lmin * nchunks + c] + run[lmin] + rank;
                node_array[pos] = (int32_t)v;
                // one rank per GPU: a halo atom's row is its FROM row here
                if (lmin == canon || (only >= 0 && o != only)) crow[v] = pos;
                cur = next_list_only(o, m, p, cur, only);
            }
            __syncwarp();
            if (lane == 0) run[lmin] += __popc(bal);
            __syncwarp();
        }
    }
}

__global__ void k_list_starts(const int32_t* __restrict__ offs, int nlists, int64_t nchunks,
                              int32_t* __restrict__ list_off) {
    int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l <= nlists) list_off[l] = offs[(int64_t)l * nchunks];  // offs[nlists*nchunks] = total
}

__global__ void k_from_src(const int32_t* __restrict__ node_array, const int32_t* __restrict__ crow,
                           const int32_t* __restrict__ from_ranges, int p, int64_t ntot,
                           const int32_t* __restrict__ from_prefix, int32_t* __restrict__ xdst,
                           int32_t* __restrict__ xsrc) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= ntot) return;
    int lo = 0, hi = p - 1;  // last i with from_prefix[i] <= k
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (from_prefix[mid] <= k) lo = mid; else hi = mid - 1;
    }
    int r = from_ranges[2 * lo] + (int)(k - from_prefix[lo]);
    xdst[k] = r;
    xsrc[k] = crow[node_array[r]];
}

__global__ void k_edge_lsrc(const int32_t* __restrict__ row, const int32_t* __restrict__ src,
                            int64_t n, const int32_t* __restrict__ owner,
                            const int32_t* __restrict__ crow, const int32_t* __restrict__ node_array,
                            const int32_t* __restrict__ list_off, int p,
                            int32_t* __restrict__ lsrc, int32_t* __restrict__ flags) {
    // 16 lanes per row (~45-edge rows fill 3 x 16 slots instead of 2 x 32)
    int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 4) + (threadIdx.x >> 4);
    if (v >= n) return;
    const int i = owner[v];
    const int stride = 1 + 2 * p;
    for (int e = row[v] + (threadIdx.x & 15); e < row[v + 1]; e += 16) {
        int u = src[e];
        int ou = owner[u];
        int r;
        if (ou == i) {
            r = crow[u];
        } else {
            int blk = i * stride + 1 + p + ou;
            int lo = list_off[blk], hi = list_off[blk + 1] - 1;
            r = -1;
            while (lo <= hi) {
                int mid = (lo + hi) >> 1;
                int x = node_array[mid];
                if (x == u) {
                    r = mid;
                    break;
                }
                if (x < u) lo = mid + 1; else hi = mid - 1;
            }
            if (r < 0) atomicOr(&flags[1], 8);
        }
        lsrc[e] = r;
    }
}

}  // namespace

size_t select_ws_bytes(int nranks) {
    (void)nranks;
    return sizeof(SelState) + (size_t)kSelMaxRanks * 256 * 4 + 256;
}

void launch_select(const double* keys, int64_t n, const int64_t* ranks_host, int nranks,
                   void* ws, double* out_dev, cudaStream_t s) {
    if (nranks <= 0) return;
    if (nranks > kSelMaxRanks) raise(kRuntime, "select: too many ranks");
    SelState st{};
    st.nr = nranks;
    st.ng = 1;
    st.ugroup[0] = 0;
    for (int k = 0; k < nranks; ++k) {
        st.prefix[k] = 0;
        st.rem[k] = ranks_host[k];
        st.gmap[k] = 0;
    }
    SelState* dst = static_cast<SelState*>(ws);
    unsigned int* hist = reinterpret_cast<unsigned int*>(static_cast<char*>(ws) + sizeof(SelState));
    GMD_CUDA(cudaMemcpyAsync(dst, &st, sizeof st, cudaMemcpyHostToDevice, s));
    GMD_CUDA(cudaMemsetAsync(hist, 0, (size_t)kSelMaxRanks * 256 * 4, s));
    const auto* k64 = reinterpret_cast<const unsigned long long*>(keys);
    int grid = (int)std::min<int64_t>(148 * 4, std::max<int64_t>(1, (n + 255) / 256));
    unsigned int* ticket = reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(hist) +
                                                           (size_t)kSelMaxRanks * 256 * 4);
    GMD_CUDA(cudaMemsetAsync(ticket, 0, 4, s));
    for (int pass = 0; pass < 8; ++pass) {
        const int shift = 56 - 8 * pass;
        k_sel_pass<<<grid, 256, 0, s>>>(k64, n, dst, hist, ticket, shift, out_dev, pass == 7 ? 1 : 0);
        GMD_LAUNCH_CHECK();
    }
}

void launch_owner(const double* fw_axis, int64_t n, const Bounds& bd, int32_t* owner,
                  cudaStream_t s) {
    k_owner<<<div_up(n, 256), 256, 0, s>>>(fw_axis, n, bd, owner);
    GMD_LAUNCH_CHECK();
}

void launch_required(const int32_t* row, const int32_t* src, int64_t n, const int32_t* owner,
                     unsigned long long* req, cudaStream_t s) {
    k_required<<<div_up(n, 8), 256, 0, s>>>(row, src, n, owner, req);
    GMD_LAUNCH_CHECK();
}

int64_t layout_chunks(int64_t nid) { return (nid + kChunk - 1) / kChunk; }
int64_t layout_nlists(int p) { return (int64_t)p * (1 + 2 * p); }

void launch_layout_plan(const int32_t* owner, const unsigned long long* req, int64_t nid, int p,
                        LayoutWs& ws, int32_t* list_off, int only, cudaStream_t s) {
    const int nlists = (int)layout_nlists(p);
    const int64_t nch = layout_chunks(nid);
    const size_t sm = (size_t)nlists * 4;
    if (nch > 0) {
        k_lay_count<<<(unsigned)nch, 32, sm, s>>>(owner, req, nid, p, nlists, nch, ws.counts, only);
        GMD_LAUNCH_CHECK();
    } else {
        GMD_CUDA(cudaMemsetAsync(ws.counts, 0, sizeof(int32_t) * (nlists + 1), s));
    }
    exclusive_scan_i32(ws.counts, ws.counts, (int64_t)nlists * nch, ws.scan_tmp,
                       ws.scan_tmp_bytes, s);
    k_list_starts<<<div_up(nlists + 1, 256), 256, 0, s>>>(ws.counts, nlists, nch > 0 ? nch : 0,
                                                          list_off);
    GMD_LAUNCH_CHECK();
}

void launch_layout_fill(const int32_t* owner, const unsigned long long* req, int64_t nid, int p,
                        LayoutWs& ws, int32_t* node_array, int32_t* crow, int only,
                        cudaStream_t s) {
    const int nlists = (int)layout_nlists(p);
    const int64_t nch = layout_chunks(nid);
    const size_t sm = (size_t)nlists * 4;
    if (nch > 0) {
        k_lay_scatter<<<(unsigned)nch, 32, sm, s>>>(owner, req, nid, p, nlists, nch, ws.counts,
                                                     node_array, crow, only);
        GMD_LAUNCH_CHECK();
    }
}

void launch_required_rank(const int32_t* row, const int32_t* src, int64_t n, const int32_t* owner,
                          int r, unsigned long long* req, cudaStream_t s) {
    k_required_rank<<<div_up(n, 8), 256, 0, s>>>(row, src, n, owner, r, req);
    GMD_LAUNCH_CHECK();
}

void launch_owned_flags(const int32_t* owner, int64_t n, int r, int32_t* flag, cudaStream_t s) {
    k_flag_owned<<<div_up(n, 256), 256, 0, s>>>(owner, n, r, flag);
    GMD_LAUNCH_CHECK();
}

void launch_owned_compact(const int32_t* owner, int64_t n, int r, const int32_t* pos,
                          int32_t* nodes, cudaStream_t s) {
    k_compact_owned<<<div_up(n, 256), 256, 0, s>>>(owner, n, r, pos, nodes);
    GMD_LAUNCH_CHECK();
}

void launch_flag_interior(int64_t n_own, const int32_t* nodes, const int32_t* row, const int32_t* src,
                          const int32_t* owner, int r, int32_t* flag, cudaStream_t s) {
    if (n_own <= 0) return;
    k_flag_interior<<<div_up(n_own, 256), 256, 0, s>>>(n_own, nodes, row, src, owner, r, flag);
    GMD_LAUNCH_CHECK();
}

void launch_split_nodes(int64_t n_own, const int32_t* nodes, const int32_t* pos, int32_t* out,
                        cudaStream_t s) {
    if (n_own <= 0) return;
    k_split_nodes<<<div_up(n_own, 256), 256, 0, s>>>(n_own, nodes, pos, out);
    GMD_LAUNCH_CHECK();
}

void launch_send_rows(int32_t t0, int32_t t1, const int32_t* node_array, const int32_t* crow,
                      int32_t* xsend, cudaStream_t s) {
    if (t1 <= t0) return;
    k_send_rows<<<div_up(t1 - t0, 256), 256, 0, s>>>(t0, t1, node_array, crow, xsend);
    GMD_LAUNCH_CHECK();
}

void launch_from_src(const int32_t* node_array, const int32_t* crow, const int32_t* from_ranges,
                     int p, int64_t nfrom_total, const int32_t* from_prefix, int32_t* xdst,
                     int32_t* xsrc, cudaStream_t s) {
    if (nfrom_total == 0) return;
    k_from_src<<<div_up(nfrom_total, 256), 256, 0, s>>>(node_array, crow, from_ranges, p,
                                                         nfrom_total, from_prefix, xdst, xsrc);
    GMD_LAUNCH_CHECK();
}

void launch_edge_lsrc(const int32_t* row, const int32_t* src, int64_t n, const int32_t* owner,
                      const int32_t* crow, const int32_t* node_array, const int32_t* list_off,
                      int p, int32_t* lsrc, int32_t* flags, cudaStream_t s) {
    k_edge_lsrc<<<div_up(n, 16), 256, 0, s>>>(row, src, n, owner, crow, node_array, list_off, p,
                                             lsrc, flags);
    GMD_LAUNCH_CHECK();
}

}  // namespace gmd
