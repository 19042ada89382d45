// Inter-stage P2P over NVLink 5 (K9 of DESIGN.md). Each receiving stage
// registers its activation / gradient ring once (CUDA IPC handles exchanged
// over torch.distributed at init); senders map the peer ring and write into
// it with an SM-driven copy kernel (16-byte vector stores over NVLink), then
// record an interprocess event the receiver's compute stream waits on —
// no host staging, no NCCL on the pipeline path. Replaces the modeled,
// serialized link of send() (sp/engine/py_kernel.py:184-214).
#include <cstring>

#include "common.cuh"

namespace vp {
namespace {

__global__ void __launch_bounds__(512) put_kernel(uint4* __restrict__ dst,
                                                  const uint4* __restrict__ src, int64_t n16) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  // 4 independent 16-byte loads in flight per thread before the stores.
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < n16; i += stride) dst[i] = src[i];
}

__global__ void put_tail_kernel(uint8_t* dst, const uint8_t* src, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[i];
}

}  // namespace
}  // namespace vp

using namespace vp;

extern "C" int vp_device_alloc(int64_t bytes, void** ptr_out) {
  if (bytes <= 0 || !ptr_out) return VP_ERR_ARGS;
  return cudaMalloc(ptr_out, static_cast<size_t>(bytes));
}
extern "C" int vp_device_free(void* ptr) { return cudaFree(ptr); }

extern "C" int vp_ipc_get_mem_handle(void* dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out) return VP_ERR_ARGS;
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, dev_ptr);
  if (e != cudaSuccess) return e;
  static_assert(sizeof(h) <= VP_IPC_HANDLE_BYTES, "handle size");
  std::memcpy(handle_out, &h, sizeof(h));
  return VP_OK;
}

extern "C" int vp_ipc_open_mem_handle(const void* handle, void** dev_ptr_out) {
  if (!handle || !dev_ptr_out) return VP_ERR_ARGS;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  return cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
}

extern "C" int vp_ipc_close_mem_handle(void* dev_ptr) { return cudaIpcCloseMemHandle(dev_ptr); }

extern "C" int vp_ipc_event_create(void** event_out, void* handle_out) {
  if (!event_out || !handle_out) return VP_ERR_ARGS;
  cudaEvent_t ev;
  cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming | cudaEventInterprocess);
  if (e != cudaSuccess) return e;
  cudaIpcEventHandle_t h;
  e = cudaIpcGetEventHandle(&h, ev);
  if (e != cudaSuccess) return e;
  std::memcpy(handle_out, &h, sizeof(h));
  *event_out = ev;
  return VP_OK;
}

extern "C" int vp_ipc_event_open(const void* handle, void** event_out) {
  if (!handle || !event_out) return VP_ERR_ARGS;
  cudaIpcEventHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  cudaEvent_t ev;
  cudaError_t e = cudaIpcOpenEventHandle(&ev, h);
  if (e != cudaSuccess) return e;
  *event_out = ev;
  return VP_OK;
}

extern "C" int vp_event_destroy(void* event) {
  return cudaEventDestroy(reinterpret_cast<cudaEvent_t>(event));
}
extern "C" int vp_event_record(void* event, void* stream) {
  return cudaEventRecord(reinterpret_cast<cudaEvent_t>(event),
                         reinterpret_cast<cudaStream_t>(stream));
}
extern "C" int vp_stream_wait_event(void* stream, void* event) {
  return cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream),
                             reinterpret_cast<cudaEvent_t>(event), 0);
}
extern "C" int vp_event_query(void* event) {
  cudaError_t e = cudaEventQuery(reinterpret_cast<cudaEvent_t>(event));
  if (e == cudaSuccess) return 0;
  if (e == cudaErrorNotReady) return 1;
  return e;
}

extern "C" int vp_p2p_put(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes < 0 || (!dst && bytes) || (!src && bytes)) return VP_ERR_ARGS;
  if (bytes == 0) return VP_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool aligned =
      ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
  int64_t n16 = aligned ? bytes / 16 : 0;
  if (n16) {
    // Enough CTAs to saturate NVLink without occupying the whole chip.
    const int64_t want = (n16 + 511) / 512;
    const unsigned grid = static_cast<unsigned>(want < 64 ? want : 64);
    put_kernel<<<grid, 512, 0, st>>>(reinterpret_cast<uint4*>(dst),
                                     reinterpret_cast<const uint4*>(src), n16);
  }
  const int64_t done = n16 * 16, rest = bytes - done;
  if (rest > 0)
    put_tail_kernel<<<static_cast<unsigned>((rest + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<uint8_t*>(dst) + done, reinterpret_cast<const uint8_t*>(src) + done, rest);
  return launch_status();
}
