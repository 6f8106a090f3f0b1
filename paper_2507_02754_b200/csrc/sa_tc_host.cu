// sa_tc_host.cu -- host helpers for the tensor-core kernels: TMA tensor-map encoding through the
// driver entry point (no libcuda link dependency) and the bf16 -> fp16 operand conversion pass.
#include <cudaTypedefs.h>

#include <mutex>

#include "sa_tc_common.cuh"

namespace sa {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool make_tmap_bnhd_f16(CUtensorMap* m, const void* base, int B, int rows, int H, int D, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {cuuint64_t(D), cuuint64_t(H), cuuint64_t(rows), cuuint64_t(B)};
  cuuint64_t strides[3] = {cuuint64_t(D) * 2, cuuint64_t(D) * H * 2, cuuint64_t(D) * H * rows * 2};
  cuuint32_t box[4] = {cuuint32_t(D < 64 ? D : 64), 1, cuuint32_t(box_rows), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Row-staging map over a [B, rows, HD] tensor of 16-bit elements (HD = heads x D): box of (D + 8)
// elements x box_rows rows, no swizzle, so a copy lands as rows of pitch D + 8 elements -- the
// padded pitch the kernels' row-per-thread reads are bank-conflict free with.  The 8 extra columns
// belong to the next head (or fall outside the row: zero fill) and are never read.
bool make_tmap_rows_pitched(CUtensorMap* m, const void* base, int B, int rows, int HD, int D, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {cuuint64_t(HD), cuuint64_t(rows), cuuint64_t(B), 1};
  cuuint64_t strides[3] = {cuuint64_t(HD) * 2, cuuint64_t(HD) * rows * 2, cuuint64_t(HD) * rows * B * 2};
  cuuint32_t box[4] = {cuuint32_t(D + 8), cuuint32_t(box_rows), 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                  // no L2 promotion: the 8 padding columns touch the next head's row, which a 256-byte
                  // promotion would pull from DRAM whole (+43% bwd_q traffic at the memory-bound point)
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

namespace {
// bf16 -> fp16, 8 elements per thread-iteration.  Exact for |x| in the fp16 normal range; the
// MMA operands must share one 16-bit format.
__global__ void __launch_bounds__(256) cvt_bf16_f16(const uint4* __restrict__ a, uint4* __restrict__ ao, int64_t na8,
                                                    const uint4* __restrict__ b, uint4* __restrict__ bo, int64_t nb8) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < na8 + nb8; t += int64_t(gridDim.x) * blockDim.x) {
    const uint4* src = t < na8 ? a + t : b + (t - na8);
    uint4* dst = t < na8 ? ao + t : bo + (t - na8);
    uint4 x = __ldg(src);
    uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 f = tc::bf16x2_to_f2(w[e]);
      w[e] = tc::pack_f16x2(f.x, f.y);
    }
    *dst = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

}  // namespace

// bf16 -> fp16 copies of two tensors of na and nb elements (multiples of 8), one launch.
cudaError_t convert_two_f16(const void* a, void* ao, int64_t na, const void* b, void* bo, int64_t nb, int num_sms,
                            cudaStream_t st) {
  const int64_t na8 = na / 8, nb8 = nb / 8;
  int blocks = int((na8 + nb8 + 255) / 256);
  if (blocks > num_sms * 8) blocks = num_sms * 8;
  if (blocks < 1) blocks = 1;
  KernelScope ks("tc_cvt_f16", st);
  cvt_bf16_f16<<<blocks, 256, 0, st>>>((const uint4*)a, (uint4*)ao, na8, (const uint4*)b, (uint4*)bo, nb8);
  return cudaGetLastError();
}

cudaError_t convert_pair_f16(const void* a, void* ao, const void* b, void* bo, int64_t n, int num_sms,
                             cudaStream_t st) {
  return convert_two_f16(a, ao, n, b, bo, n, num_sms, st);
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace sa
