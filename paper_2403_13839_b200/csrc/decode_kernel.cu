// decode_kernel.cu -- the sm_100a decode kernel (disasm.py:71-172) and its
// launcher, compiled as its own object so it can be tuned without rebuilding
// the decompile kernel (upy.cu).
#include <cuda_runtime.h>
#include "decode.h"

// One warp per object (grid-stride); tables and record staging in shared memory.
// Software-pipelined: while a warp decodes object o, the header of o + 2*stride
// and the first 512 code bytes of o + stride are already in flight.
__device__ __forceinline__ void obj_hdr(const upy_arena& A, i64 x, u64* off, u32* len, u32* minor) {
  if (x < A.n_objs) {
    const upy_obj* ob = &A.objs[x];
    *off = ob->code_off;
    *len = ob->code_len;
    *minor = ob->minor;
  } else {
    *off = 0;
    *len = 0;
    *minor = 0;
  }
}
__device__ __forceinline__ uint4 first_chunk(const upy_arena& A, u64 off, u32 len, u32 minor, int lane) {
  if (minor >= 8 && minor <= 10 && !(len & 1) && 8u * lane < (len >> 1))
    return *reinterpret_cast<const uint4*>(A.bytes + off + 16 * lane);
  return make_uint4(0, 0, 0, 0);
}
__global__ void __launch_bounds__(256, 2) upy_decode_kernel(upy_arena A, upy_ins* __restrict__ ins,
                                                            upy_decoded* __restrict__ dec) {
  const int lane = threadIdx.x & 31;
  const i64 warp = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  __shared__ u32 tab[3][256];              // 3.8-3.10 opcode tables
  __shared__ __align__(16) upy_ins stage[256 / 32][256];  // per-warp record staging (24 KB)
  for (int i = threadIdx.x; i < 3 * 256; i += blockDim.x) tab[i >> 8][i & 255] = UPY_OPTABLE_DEV[i >> 8][i & 255];
  __syncthreads();
  upy_ins* my_stage = stage[threadIdx.x >> 5];
  u64 off0, off1, off2;
  u32 len0, len1, len2, min0, min1, min2;
  obj_hdr(A, warp, &off0, &len0, &min0);
  uint4 w0 = first_chunk(A, off0, len0, min0, lane);
  obj_hdr(A, warp + nwarps, &off1, &len1, &min1);
  for (i64 o = warp; o < A.n_objs; o += nwarps) {
    uint4 w1 = first_chunk(A, off1, len1, min1, lane);
    obj_hdr(A, o + 2 * nwarps, &off2, &len2, &min2);
    const u8* code = A.bytes + off0;
    upy_ins* rec = ins + (off0 >> 1);
    int minor = (int)min0;
    if (minor >= 8 && minor <= 10) {
      decode_warp(code, len0, minor, rec, &dec[o], tab[minor - 8], my_stage, w0);
    } else if (lane == 0) {
      if (minor == 11) {
        decode_scalar(code, len0, minor, rec, &dec[o]);
      } else {
        dec[o].status = UPY_ST_INTERNAL;
        dec[o].n_instrs = 0;
      }
    }
    __syncwarp();
    off0 = off1, len0 = len1, min0 = min1, w0 = w1;
    off1 = off2, len1 = len2, min1 = min2;
  }
}

// Launcher used by upy_decode_batch (upy.cu); returns the launch error.
cudaError_t upy_decode_launch(const upy_arena* arena, upy_ins* ins, upy_decoded* dec, cudaStream_t s, int sms) {
  const int threads = 256;
  i64 blocks = (arena->n_objs * 32 + threads - 1) / threads;
  i64 max_blocks = (i64)sms * 64;
  if (blocks > max_blocks) blocks = max_blocks;
  upy_decode_kernel<<<(unsigned)blocks, threads, 0, s>>>(*arena, ins, dec);
  return cudaGetLastError();
}
