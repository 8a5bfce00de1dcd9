// Uᵀ built on the device from the uploaded U (scfr_create, unsharded
// handles): the reference's `CsrMatrix.transposed()` (pkg/kernels.py:95-127,
// via pkg/operators.py:164-180) is a stable transpose, so column c of U
// becomes row c of Uᵀ with its entries in increasing row order and the same
// fp64 values.  A stable LSD radix sort of U's entry ids keyed by column
// gives exactly that order, so the result is bit-identical to the caller's
// Uᵀ for every bundle the reference builds, and the caller's Uᵀ arrays need
// not be read, converted and copied on the host (a quarter of create's host
// memory traffic on Goofspiel-5).  Spot checks against the caller's Uᵀ
// (shape, nnz, 64 row pointers and 64 entries spread over the matrix) catch
// a Uᵀ that is not U's transpose; SCFR_HOST_UT=1 uploads the caller's
// instead (and the row-sharded mode always does).

#include <cstring>
#include <vector>

#include <cub/cub.cuh>

#include "runtime.h"

namespace scfr {

__global__ void k_entry_rows(int rows, const int* __restrict__ indptr, int* __restrict__ row_of) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    for (int k = indptr[r], e = indptr[r + 1]; k < e; ++k) row_of[k] = r;
}

__global__ void k_col_counts(int nnz, const int* __restrict__ col, int* __restrict__ cnt) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < nnz) atomicAdd(cnt + col[k], 1);
}

__global__ void k_seq(int n, int* __restrict__ v) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) v[k] = k;
}

// Entry i of Uᵀ (column-major order of U) is U's entry perm[i].
__global__ void k_transpose_gather(int nnz, const int* __restrict__ perm, const int* __restrict__ row_of,
                                   const double* __restrict__ data, int* __restrict__ tix,
                                   double* __restrict__ tdata) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nnz) return;
    const int k = perm[i];
    tix[i] = row_of[k];
    tdata[i] = data[k];
}

__global__ void k_round_f32(int n, const double* __restrict__ d, float* __restrict__ f) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) f[i] = __double2float_rn(d[i]);
}

__global__ void k_gather_i32(int n, const int* __restrict__ src, const int* __restrict__ at, int* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = src[at[i]];
}
__global__ void k_gather_pairs(int n, const int* __restrict__ ix, const double* __restrict__ d,
                               const int* __restrict__ at, int* __restrict__ oix, double* __restrict__ od) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        oix[i] = ix[at[i]];
        od[i] = d[at[i]];
    }
}

void derive_transpose(const DevCsr& U, const scfr_csr* UT, DevCsr& T, cudaStream_t s, bool f32) {
    const int rows = U.cols, cols = U.rows, nnz = U.nnz;
    if (!UT || UT->rows != rows || UT->cols != cols || UT->nnz != nnz)
        fail(SCFR_EINVAL, "the transposed payoff matrix does not have U's transposed shape");
    if (!UT->indptr || (nnz > 0 && (!UT->indices || !UT->data))) fail(SCFR_EINVAL, "csr has a NULL array");
    if (UT->indptr[0] != 0 || UT->indptr[rows] != nnz) fail(SCFR_EINVAL, "indptr must start at 0 and end at nnz");
    T.full_rows = rows;
    T.row0 = 0;
    T.chunk = rows;
    T.rows = rows;
    T.cols = cols;
    T.nnz = nnz;
    T.indptr.alloc(rows + 1);
    T.indices.alloc(std::max(nnz, 1));
    T.data.alloc(std::max(nnz, 1));
    T.indptr.zero(s);
    if (nnz > 0) {
        DevBuf<int> row_of, keys_out, perm_in, perm_out;
        row_of.alloc(nnz);
        keys_out.alloc(nnz);
        perm_in.alloc(nnz);
        perm_out.alloc(nnz);
        k_entry_rows<<<grid_for(U.rows), TPB, 0, s>>>(U.rows, U.indptr.p, row_of.p);
        k_col_counts<<<grid_for(nnz), TPB, 0, s>>>(nnz, U.indices.p, T.indptr.p + 1);  // counts at c + 1
        k_seq<<<grid_for(nnz), TPB, 0, s>>>(nnz, perm_in.p);
        CUDA_OK(cudaGetLastError());
        int bits = 1;  // keys: U's columns, [0, rows)
        while (bits < 31 && (1ll << bits) < (long long)rows) ++bits;
        size_t tb_sort = 0, tb_scan = 0;
        CUDA_OK(cub::DeviceRadixSort::SortPairs(nullptr, tb_sort, U.indices.p, keys_out.p, perm_in.p, perm_out.p,
                                                nnz, 0, bits, s));
        CUDA_OK(cub::DeviceScan::InclusiveSum(nullptr, tb_scan, T.indptr.p + 1, T.indptr.p + 1, rows, s));
        DevBuf<unsigned char> tmp;
        tmp.alloc(std::max(tb_sort, tb_scan));
        // stable: within one column, entries keep U's row-major order
        CUDA_OK(cub::DeviceRadixSort::SortPairs(tmp.p, tb_sort, U.indices.p, keys_out.p, perm_in.p, perm_out.p,
                                                nnz, 0, bits, s));
        CUDA_OK(cub::DeviceScan::InclusiveSum(tmp.p, tb_scan, T.indptr.p + 1, T.indptr.p + 1, rows, s));
        k_transpose_gather<<<grid_for(nnz), TPB, 0, s>>>(nnz, perm_out.p, row_of.p, U.data.p, T.indices.p,
                                                         T.data.p);
        CUDA_OK(cudaGetLastError());
        // spot checks against the caller's Uᵀ: 64 row pointers and 64
        // entries spread over the matrix
        constexpr int kProbe = 64;
        std::vector<int> at_r(kProbe), at_k(kProbe);
        for (int i = 0; i < kProbe; ++i) {
            at_r[i] = (int)((int64_t)rows * i / (kProbe - 1));
            at_k[i] = (int)((int64_t)(nnz - 1) * i / (kProbe - 1));
        }
        DevBuf<int> dat, dout, dix;
        DevBuf<double> dd;
        dat.alloc(2 * kProbe);
        dout.alloc(kProbe);
        dix.alloc(kProbe);
        dd.alloc(kProbe);
        CUDA_OK(copy_async(dat.p, at_r.data(), kProbe * sizeof(int), cudaMemcpyHostToDevice, s));
        CUDA_OK(copy_async(dat.p + kProbe, at_k.data(), kProbe * sizeof(int), cudaMemcpyHostToDevice, s));
        k_gather_i32<<<1, kProbe, 0, s>>>(kProbe, T.indptr.p, dat.p, dout.p);
        k_gather_pairs<<<1, kProbe, 0, s>>>(kProbe, T.indices.p, T.data.p, dat.p + kProbe, dix.p, dd.p);
        CUDA_OK(cudaGetLastError());
        std::vector<int> hp(kProbe), hix(kProbe);
        std::vector<double> hd(kProbe);
        CUDA_OK(copy_async(hp.data(), dout.p, kProbe * sizeof(int), cudaMemcpyDeviceToHost, s));
        CUDA_OK(copy_async(hix.data(), dix.p, kProbe * sizeof(int), cudaMemcpyDeviceToHost, s));
        CUDA_OK(copy_async(hd.data(), dd.p, kProbe * sizeof(double), cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        for (int i = 0; i < kProbe; ++i)
            if (UT->indptr[at_r[i]] != hp[i] || UT->indices[at_k[i]] != hix[i] ||
                std::memcmp(&UT->data[at_k[i]], &hd[i], sizeof(double)) != 0)
                fail(SCFR_EINVAL, "the transposed payoff matrix is not the transpose of U");
    }
    if (f32) {  // the iteration's copy, rounded once (as upload_csr)
        T.data32.alloc(std::max(nnz, 1));
        if (nnz) k_round_f32<<<grid_for(nnz), TPB, 0, s>>>(nnz, T.data.p, T.data32.p);
        CUDA_OK(cudaGetLastError());
    }
}

// Row pointers of a device CSR at the given rows (csr_level_info of a Uᵀ
// derived here: its level bookkeeping must come from the device copy).
void device_row_ptrs(const DevCsr& D, const std::vector<int>& rows, std::vector<int64_t>& out, cudaStream_t s) {
    out.assign(rows.size(), 0);
    if (rows.empty()) return;
    const int n = (int)rows.size();
    DevBuf<int> at, val;
    at.alloc(n);
    val.alloc(n);
    std::vector<int> hv(n);
    CUDA_OK(copy_async(at.p, rows.data(), n * sizeof(int), cudaMemcpyHostToDevice, s));
    k_gather_i32<<<(n + 127) / 128, 128, 0, s>>>(n, D.indptr.p, at.p, val.p);
    CUDA_OK(cudaGetLastError());
    CUDA_OK(copy_async(hv.data(), val.p, n * sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    for (int i = 0; i < n; ++i) out[i] = hv[i];
}

}  // namespace scfr
