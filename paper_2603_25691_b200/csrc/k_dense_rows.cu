// k_dense_rows.cu — the q-pass over DENSE rows of a 3-way plan on the FP64 tensor cores (sm_100a
// DMMA).
//
// The reference's q-pass (observations.hpp:174-198 via unaligned.hpp:110-111) adds, for every
// observation l of row i = i_k(l) with other indices (a_l, b_l),
//     Yhat(i,:) += w_l (Xhat(i,:) . z_l) z_l,      z_l = A_1(a_l,:) o A_2(b_l,:).
// Group the observations of one row by cell: W_i(a, b) = number of draws (the multiplicity of the
// coalesced plan) of cell (i, a, b), zero when the cell was never drawn.  Then, with
// U_i = A_1 diag(Xhat(i,:)) (n_1 x r),
//     S_i = U_i A_2'                 (n_1 x n_2: S_i(a, b) = Xhat(i,:) . z_(a,b))
//     T_i = W_i o S_i                (the multiplicity-weighted dots; zero off the support)
//     P_i = T_i A_2                  (n_1 x r)
//     Yhat(i, c) = sum_a A_1(a, c) P_i(a, c),
// which is the same sum, exactly (cells with W = 0 add 0 x S = 0).  A row whose cells are mostly
// drawn (the Zipf head of config 4: row 0 takes 16 % of the 1e9 draws, ~610 per cell) costs
// 2 n_1 n_2 r FMA this way — two dense GEMMs — against nnz_i x 2 r on the entry-by-entry path, so
// past a density of ~0.3 the GEMM form on DMMA wins (capi.cu build_run_parts picks the rows; the
// run kernel k_runs.cu takes the rest).  Every drawn cell is still visited once per application:
// W_i is read from HBM each time (4 B per cell), Xhat(i,:) enters through U_i.
//
// Work unit (task): one dense row i and one block of BA = 64 values of a.  A CTA of 8 warps runs
// tasks round-robin; warp w owns the 8 rows a0 + 8w .. +7 of the block (one m8 DMMA row tile) and
// walks the b axis in chunks of BB = 64:
//   GEMM 1   S(8 x 64)  = U(8 x RP) . A_2chunk(64 x RP)'     (RP/4 k-steps x 8 n-tiles)
//   scale    T = W o S                                          (W chunk: int32 multiplicities)
//   GEMM 2   P(8 x RP) += T(8 x 64) . A_2chunk(64 x RP)       (16 k-steps x RP/8 n-tiles)
// The S accumulator IS GEMM 2's A operand with no data movement: DMMA m8n8k4 leaves lane
// (g, kq) holding S(g, 8nt + 2kq + e), e = 0, 1, and an A fragment wants A(g, kq); so GEMM 2 walks
// its K axis (b) in the permuted order k-step (nt, e) <-> b = 8nt + 2kq + e and loads the B
// fragment A_2(8nt + 2kq + e, 8nc + g) to match.  A_2 chunks and W chunks are double buffered in
// shared memory by cp.async (A_2 is read from L2: 256 KB for config 4), both XOR-swizzled in 32 B
// units so that both GEMMs' fragment loads and the W loads are conflict-free (2 wavefronts per
// 256 B).  At the end of a task the warp folds Yhat's share sum_a A_1(a, c) P(a, c) over its 8
// rows (butterfly), the CTA sums its warps in order, and the last of the row's tasks to arrive sums
// the tasks' partial rows in block order and writes Yhat(i,:): fixed order, no fp64 atomics.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "kernels.cuh"

namespace cphifi {
namespace {

constexpr int DT = 256;           // threads per CTA
constexpr int DW = DT / 32;       // warps: 8 rows of a each
constexpr int BA = 8 * DW;        // a per task
constexpr int BB = 64;            // b per chunk

inline unsigned grid_for(int64_t n, int t, int cap = 8192) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + t - 1) / t, cap));
}

__device__ __forceinline__ void dmma_d(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(void* dst, const void* src, bool pred) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    const int sz = pred ? 16 : 0;  // 0: zero-fill
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// A_2 chunk: row b (BB rows) of RP doubles; the 32-byte unit u of row b sits at unit u ^ (b & 3)
template <int RP>
__device__ __forceinline__ int a2_at(int b, int c) {
    return b * RP + ((((c >> 2) ^ (b & 3))) << 2) + (c & 3);
}
// W chunk: row a (BA rows) of BB int32; the 32-byte unit u (8 ints) of row a sits at u ^ (a & 7)
__device__ __forceinline__ int w_at(int a, int b) { return a * BB + (((b >> 3) ^ (a & 7)) << 3) + (b & 7); }

template <int RP>
struct DLay {
    static constexpr size_t a2 = sizeof(double) * BB * RP;  // one A_2 chunk
    static constexpr size_t w = sizeof(int32_t) * BA * BB;  // one W chunk
    static constexpr size_t stage = a2 + w;
    static constexpr size_t red = sizeof(double) * DW * RP;
    static constexpr size_t bytes = 2 * stage + red + 16;
};

template <int RP>
__global__ void __launch_bounds__(DT, 2) dense_rows_kernel(const DenseRowsArgs p) {
    using L = DLay<RP>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* red = reinterpret_cast<double*>(smem_raw + 2 * L::stage);
    unsigned* flag = reinterpret_cast<unsigned*>(smem_raw + 2 * L::stage + L::red);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int g = lane >> 2, kq = lane & 3;
    const int nab = (int)(p.n1p / BA), nbc = (int)(p.n2p / BB);
    const int64_t ntask = (int64_t)p.nd * nab;
    const double* a1 = p.a1;
    const double* a2 = p.a2;

    // the chunk sequence of this CTA: tasks blockIdx.x, + gridDim.x, ...; nbc chunks per task
    const int64_t my_tasks = ntask > blockIdx.x ? (ntask - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t nseq = my_tasks * nbc;
    auto issue = [&](int64_t sidx) {
        const int64_t t = blockIdx.x + (sidx / nbc) * gridDim.x;
        const int bc = (int)(sidx % nbc);
        const int st = (int)(sidx & 1);
        double* sa2 = reinterpret_cast<double*>(smem_raw + st * L::stage);
        int32_t* sw = reinterpret_cast<int32_t*>(smem_raw + st * L::stage + L::a2);
        const int k = (int)(t / nab), ab = (int)(t % nab);
        const int b0 = bc * BB;
        // A_2 rows b0 .. b0 + 63 (zero beyond n_2): BB x RP / 2 pieces of 16 B
        for (int e = tid; e < BB * RP / 2; e += DT) {
            const int b = e / (RP / 2), c = 2 * (e % (RP / 2));
            const bool ok = b0 + b < p.n2;
            cp16(sa2 + a2_at<RP>(b, c), a2 + (ok ? (int64_t)(b0 + b) * RP + c : 0), ok);
        }
        // W(i_k, a0 .., b0 ..): BA x BB int32, 16 pieces of 16 B per row
        const int32_t* wsrc = p.w + ((int64_t)k * p.n1p + (int64_t)ab * BA) * p.n2p + b0;
        for (int e = tid; e < BA * BB / 4; e += DT) {
            const int a = e / (BB / 4), b = 4 * (e % (BB / 4));
            cp16(sw + w_at(a, b), wsrc + (int64_t)a * p.n2p + b, true);
        }
        cp_commit();
    };

    if (nseq > 0) issue(0);
    int64_t sidx = 0;
    for (int64_t tl = 0; tl < my_tasks; ++tl) {
        const int64_t t = blockIdx.x + tl * gridDim.x;
        const int k = (int)(t / nab), ab = (int)(t % nab);
        const int row = p.rows[k];
        const int a_me = ab * BA + 8 * w + g;  // this lane's a (A-fragment row)
        // U fragments: U(a, 4 ks + kq) = Xhat(i, c) A_1(a, c)
        double u[RP / 4];
        {
            const double* xr = p.xhat_rm + (int64_t)row * RP;
            const double* ar = a1 + (int64_t)a_me * RP;
            const bool ok = a_me < p.n1;
#pragma unroll
            for (int ks = 0; ks < RP / 4; ++ks) u[ks] = ok ? __ldg(xr + 4 * ks + kq) * __ldg(ar + 4 * ks + kq) : 0.0;
        }
        double pacc[RP / 8][2];
#pragma unroll
        for (int j = 0; j < RP / 8; ++j) pacc[j][0] = pacc[j][1] = 0.0;

        for (int bc = 0; bc < nbc; ++bc, ++sidx) {
            if (sidx + 1 < nseq) {
                issue(sidx + 1);
                cp_wait1();
            } else {
                cp_wait0();
            }
            __syncthreads();  // chunk sidx landed for every thread's copies
            const int st = (int)(sidx & 1);
            const double* sa2 = reinterpret_cast<const double*>(smem_raw + st * L::stage);
            const int32_t* sw = reinterpret_cast<const int32_t*>(smem_raw + st * L::stage + L::a2);
            // GEMM 1: S(g, 8nt + 2kq + e) over k = c
            double s[8][2];
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) s[nt][0] = s[nt][1] = 0.0;
#pragma unroll
            for (int ks = 0; ks < RP / 4; ++ks) {
#pragma unroll
                for (int nt = 0; nt < 8; ++nt) dmma_d(s[nt], u[ks], sa2[a2_at<RP>(8 * nt + g, 4 * ks + kq)]);
            }
            // T = W o S
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
                const int2 m = *reinterpret_cast<const int2*>(sw + w_at(8 * w + g, 8 * nt + 2 * kq));
                s[nt][0] *= (double)m.x;
                s[nt][1] *= (double)m.y;
            }
            // GEMM 2: P(g, 8nc + 2kq + e) += sum_b T(g, b) A_2(b, c), k-step (nt, e): b = 8nt + 2kq + e
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int b = 8 * nt + 2 * kq + e;
#pragma unroll
                    for (int nc = 0; nc < RP / 8; ++nc) dmma_d(pacc[nc], s[nt][e], sa2[a2_at<RP>(b, 8 * nc + g)]);
                }
            }
            __syncthreads();  // stage st free for the copy issued at the next chunk
        }
        // Yhat share of this warp: sum over its 8 rows a of A_1(a, c) P(a, c)
        {
            const bool ok = a_me < p.n1;
            const double* ar = a1 + (int64_t)a_me * RP;
#pragma unroll
            for (int nc = 0; nc < RP / 8; ++nc) {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int c = 8 * nc + 2 * kq + e;
                    double v = ok ? pacc[nc][e] * __ldg(ar + c) : 0.0;
                    v += __shfl_xor_sync(0xffffffffu, v, 4);
                    v += __shfl_xor_sync(0xffffffffu, v, 8);
                    v += __shfl_xor_sync(0xffffffffu, v, 16);
                    if (g == 0) red[w * RP + c] = v;
                }
            }
        }
        __syncthreads();
        double* part = p.partial + ((int64_t)k * nab + ab) * RP;
        if (tid < RP) {
            double v = red[tid];
#pragma unroll
            for (int ww = 1; ww < DW; ++ww) v += red[ww * RP + tid];
            part[tid] = v;
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            unsigned old;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(p.cnt + k) : "memory");
            const unsigned last = old == (unsigned)nab - 1;
            if (last) p.cnt[k] = 0;
            *flag = last;
        }
        __syncthreads();
        if (*flag) {  // every block of the row is in: Yhat(i,:) = sum over blocks in block order
            const double* pr = p.partial + (int64_t)k * nab * RP;
            if (tid < RP) {
                double v = __ldcg(pr + tid);
                for (int j = 1; j < nab; ++j) v += __ldcg(pr + (int64_t)j * RP + tid);
                p.yhat_rm[(int64_t)row * RP + tid] = v;
            }
        }
        __syncthreads();  // red / flag reused by the next task
    }
}

template <int RP>
void launch_dense(const DenseRowsArgs& a, int num_sms, cudaStream_t s) {
    auto kern = dense_rows_kernel<RP>;
    func_attr_once((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DLay<RP>::bytes);
    const int64_t ntask = (int64_t)a.nd * (a.n1p / BA);
    const int grid = (int)std::min<int64_t>(ntask, 2 * (int64_t)num_sms);
    kern<<<grid, DT, DLay<RP>::bytes, s>>>(a);
    CPHIFI_CHECK_LAUNCH();
}

__global__ void dense_grid_kernel(const int32_t* idx, int64_t ldq, const int32_t* mult, const int32_t* rows,
                                  const int32_t* slot, int64_t q, int64_t n1p, int64_t n2p, int32_t* w) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < q; l += (int64_t)gridDim.x * blockDim.x) {
        const int k = slot[rows[l]];
        if (k < 0) continue;
        const int32_t m = mult ? mult[l] : 1;
        atomicAdd(w + ((int64_t)k * n1p + idx[l]) * n2p + idx[ldq + l], m);
    }
}

__global__ void sum_i32_kernel(const int32_t* v, int64_t q, unsigned long long* out) {
    unsigned long long acc = 0;
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < q; l += (int64_t)gridDim.x * blockDim.x)
        acc += (unsigned long long)v[l];
    for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

__global__ void dense_key_kernel(const int32_t* rows, const int32_t* slot, int64_t q, int32_t offset, int32_t* key) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < q; l += (int64_t)gridDim.x * blockDim.x)
        if (slot[rows[l]] >= 0) key[l] += offset;
}

}  // namespace

int dense_rows_block_a() { return BA; }
int dense_rows_block_b() { return BB; }
bool dense_rows_supported(int64_t rp, int dother) { return dother == 2 && (rp == 16 || rp == 32 || rp == 64); }

void dense_rows_qpass(const DenseRowsArgs& a, int num_sms, cudaStream_t s) {
    if (a.nd <= 0) return;
    if (a.n1p % BA || a.n2p % BB) throw_invalid("dense rows: grid not padded to the block sizes");
    switch (a.rp) {
        case 16: launch_dense<16>(a, num_sms, s); break;
        case 32: launch_dense<32>(a, num_sms, s); break;
        case 64: launch_dense<64>(a, num_sms, s); break;
        default: throw_invalid("dense rows: padded rank must be 16, 32 or 64");
    }
}

void dense_grid_build(const int32_t* idx, int64_t ldq, const int32_t* mult, const int32_t* rows, const int32_t* slot,
                      int64_t q, int64_t n1p, int64_t n2p, int32_t* w, cudaStream_t s) {
    if (q == 0) return;
    dense_grid_kernel<<<grid_for(q, 256), 256, 0, s>>>(idx, ldq, mult, rows, slot, q, n1p, n2p, w);
    CPHIFI_CHECK_LAUNCH();
}

void sum_i32(const int32_t* v, int64_t q, unsigned long long* out, cudaStream_t s) {
    if (q == 0) return;
    sum_i32_kernel<<<grid_for(q, 256, 1024), 256, 0, s>>>(v, q, out);
    CPHIFI_CHECK_LAUNCH();
}

void dense_key(const int32_t* rows, const int32_t* slot, int64_t q, int32_t dense_key_value, int32_t* key,
               cudaStream_t s) {
    if (q == 0) return;
    dense_key_kernel<<<grid_for(q, 256), 256, 0, s>>>(rows, slot, q, dense_key_value, key);
    CPHIFI_CHECK_LAUNCH();
}

}  // namespace cphifi
