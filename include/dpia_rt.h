/* libdpia_rt -- C-ABI runtime of the DPIA CUDA backend (B200 / sm_100a).
 *
 * This library is the drop-in boundary that replaces the reference's
 * execution stand-in.  The reference has no native code at all: its kernels
 * are OpenCL text (emit_kernel, SRC/opencl.py:265-314) "executed" by a
 * sequential Python work-item simulator (simulate_kernel,
 * SRC/opencl.py:397-472).  The Python host binds these entry points with
 * ctypes (paper_1710_08332_b200/runtime.py); a maintainer of the reference
 * would add the same binding next to opencl.py.
 *
 * Conventions: every function returns 0 on success, otherwise a CUresult /
 * nvrtcResult / ncclResult_t code (or -1 for argument errors) and stores a
 * message readable with dpia_last_error() (thread-local).  Device pointers are
 * plain 64-bit integers; no torch (or any other framework) types appear.
 */
#ifndef DPIA_RT_H
#define DPIA_RT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- errors / devices ------------------------------------------------- */
const char* dpia_last_error(void);
/* Retain and bind the primary context of `device` (replaces nothing in the
 * reference: simulate_kernel needs no device). */
int dpia_init(int device);
int dpia_device_count(int* count);
/* attr is a CUdevice_attribute value (e.g. 16 = multiprocessor count). */
int dpia_device_attribute(int device, int attr, int* value);
int dpia_device_name(int device, char* buf, int len);

/* ---- compilation (replaces emit_kernel's text-only OpenCL output,
 *      SRC/opencl.py:265-314, with a real sm_100a binary) --------------- */
/* NVRTC version the runtime compiles with (the toolkit's libnvrtc, loaded by
   absolute path so an older libnvrtc already in the process is not used). */
int dpia_nvrtc_version(int* major, int* minor);
/* NVRTC: CUDA C source -> cubin for `arch` (e.g. "sm_100a").  `options` is a
 * '\n'-separated list of extra NVRTC flags.  On success *image points to a
 * malloc'ed cubin of *size bytes (release with dpia_free_host).  The compile
 * log (warnings or errors) is copied into log[0..logcap). */
int dpia_compile(const char* source, const char* program_name, const char* arch,
                 const char* options, void** image, size_t* size, char* log, size_t logcap);
int dpia_module_load(int device, const void* image, void** module);
int dpia_module_unload(void* module);
int dpia_get_kernel(void* module, const char* name, void** function);
/* Opt into > 48 KiB of dynamic shared memory for `function`. */
int dpia_kernel_set_smem(void* function, int bytes);
int dpia_kernel_attribute(void* function, int attr, int* value);

/* ---- memory ------------------------------------------------------------ */
int dpia_malloc(int device, size_t bytes, uint64_t* dptr);
int dpia_free(int device, uint64_t dptr);
int dpia_host_alloc(size_t bytes, void** ptr); /* pinned */
int dpia_host_free(void* ptr);
void dpia_free_host(void* ptr); /* plain free() for buffers this library malloc'ed */
int dpia_memcpy_htod(int device, uint64_t dst, const void* src, size_t bytes, void* stream);
int dpia_memcpy_dtoh(int device, void* dst, uint64_t src, size_t bytes, void* stream);
int dpia_memcpy_dtod(int device, uint64_t dst, uint64_t src, size_t bytes, void* stream);
/* pitched copies (height rows of width bytes; row r at src + r*spitch, dst + r*dpitch),
 * asynchronous on stream: used by the tile pipeline to move column panels of
 * row-major host matrices (no reference counterpart) */
int dpia_memcpy2d_htod(int device, uint64_t dst, size_t dpitch, const void* src, size_t spitch,
                       size_t width, size_t height, void* stream);
int dpia_memcpy2d_dtoh(int device, void* dst, size_t dpitch, uint64_t src, size_t spitch,
                       size_t width, size_t height, void* stream);
/* TMA descriptor (CUtensorMap, 128 bytes at out) of a row-major matrix of
 * elem_bytes (4: fp32, 8: int64) elements, rows x cols with a row pitch in
 * bytes, read in boxes of box_rows x box_cols; swizzle 0 (plain) or 128
 * (128-byte rows, 16-byte chunks XOR row % 8): the kernel parameter of an
 * emitted toLocal k-tile, work-item row fold or row store moved by
 * cp.async.bulk.tensor.2d (no reference counterpart: the reference has no
 * device code).  _f32: the plain fp32 form (tools/mmtma.py). */
int dpia_tensor_map_2d(void* out, int elem_bytes, uint64_t base, uint64_t rows, uint64_t cols,
                       uint64_t pitch, unsigned box_rows, unsigned box_cols, int swizzle);
int dpia_tensor_map_2d_f32(void* out, uint64_t base, uint64_t rows, uint64_t cols, uint64_t pitch,
                           unsigned box_rows, unsigned box_cols);
int dpia_memset(int device, uint64_t dst, int value, size_t bytes, void* stream);

/* ---- execution (replaces simulate_kernel, SRC/opencl.py:397-472) ------- */
/* cuLaunchKernel: grid (gx, gy), block (bx, by), `smem` bytes of dynamic
 * shared memory, `args` = array of pointers to each argument value. */
int dpia_launch(void* function, int device, unsigned gx, unsigned gy, unsigned bx, unsigned by,
                unsigned smem, void** args, void* stream);
/* the same with programmatic dependent launch allowed (cuLaunchKernelEx,
 * CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION): the kernel may
 * start before the previous kernel on the stream finishes and waits for it
 * with griddepcontrol.wait; used for the later phases of multi-kernel
 * programs (no reference counterpart: the reference simulator has no launches) */
int dpia_launch_pdl(void* function, int device, unsigned gx, unsigned gy, unsigned bx, unsigned by,
                    unsigned smem, void** args, void* stream);
int dpia_stream_create(int device, void** stream);
int dpia_stream_destroy(void* stream);
int dpia_stream_sync(void* stream);
int dpia_device_sync(int device);
int dpia_event_create(int device, void** event);
int dpia_event_destroy(void* event);
int dpia_event_record(void* event, void* stream);
int dpia_event_elapsed(void* start, void* stop, float* ms);
/* Make `stream` wait for `event` (cross-stream ordering of copy / compute). */
int dpia_stream_wait_event(void* stream, void* event);
/* Evict L2: overwrite a device buffer of 2x the L2 capacity on `stream`. */
int dpia_l2_flush(int device, void* stream);
/* Fill dptr[0..count) (float) with x_i = lo + (hi-lo) * h(seed, offset+i), h a
 * counter hash with 24-bit resolution -- reproducible on the host by
 * oracle/blas_np.py for any shard. */
int dpia_fill_hash_f32(int device, uint64_t dptr, uint64_t count, uint64_t offset, uint32_t seed,
                       float lo, float hi, void* stream);

/* ---- multi-GPU (NCCL, loaded at run time from the torch wheel) ---------- */
/* Peer mailboxes for the fused cross-GPU combine (emit_cuda(..., peer=True)):
 * a zeroed device allocation exported as a 64-byte CUDA IPC handle, and the
 * mapping of a peer's handle into this device's context (NVLink P2P, peer
 * access enabled lazily).  Replaces ncclAllReduce of the per-rank partials
 * with stores into every peer's mailbox from the kernel. */
int dpia_ipc_alloc(int device, size_t bytes, uint64_t* dptr, char handle[64]);
int dpia_ipc_open(int device, const char handle[64], uint64_t* dptr);
int dpia_ipc_close(int device, uint64_t dptr);

int dpia_nccl_available(void);
/* 128-byte ncclUniqueId, produced on rank 0 and broadcast by the caller. */
int dpia_nccl_unique_id(char out[128]);
int dpia_nccl_init(int device, int nranks, int rank, const char id[128]);
/* In-place sum all-reduce of `count` elements; dtype 0 = f32, 1 = f64, 2 = i64. */
int dpia_nccl_allreduce(uint64_t dptr, size_t count, int dtype, void* stream);
int dpia_nccl_destroy(void);

#ifdef __cplusplus
}
#endif
#endif /* DPIA_RT_H */
