// sd_host.cu — host-buffer (end-to-end) path of the C ABI.
//
// A plan owns kBuf device staging slots and kBuf streams on one device.
// sd_eig3_f64_host splits the batch into chunks; chunk i goes through slot
// i % kBuf on stream i % kBuf as H2D copy -> kernel -> D2H copy.  Stream
// ordering makes slot reuse safe, and three slots let the H2D of chunk i+2,
// the kernel of chunk i+1 and the D2H of chunk i run at the same time, so
// with pinned host memory the whole call is bounded by max(H2D, D2H) link
// time rather than their sum plus compute.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <new>

#include "../../include/symdiag_b200.h"

extern "C" void sd_internal_set_error(const char* msg);  // symdiag_b200.cu

namespace {
constexpr int kBuf = 3;
}  // namespace

struct sd_plan {
  int device = 0;
  int64_t chunk = 0;
  cudaStream_t stream[kBuf] = {};
  void* in[kBuf] = {};    // chunk * 6 doubles
  void* lam[kBuf] = {};   // chunk * 3 doubles
  void* ang[kBuf] = {};   // chunk * 3 doubles
  uint8_t* st[kBuf] = {};  // chunk bytes
};

namespace {

int herr(int code, const char* what, cudaError_t e) {
  char buf[512];
  snprintf(buf, sizeof buf, "%s: %s", what, e == cudaSuccess ? "" : cudaGetErrorString(e));
  sd_internal_set_error(buf);
  return code;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Generic chunked pipeline.  Tin/Tout: element types; win/wout: values per
// row of the input / each of the two outputs.
template <typename Tin, typename Tout, typename Launch>
int run_pipeline(sd_plan* plan, const Tin* A, int64_t n, int win, Tout* out0, int w0,
                 Tout* out1, int w1, uint8_t* status, Launch launch) {
  if (!plan || n < 0 || (n > 0 && (!A || !out0 || !out1 || !status)))
    return herr(SD_EINVAL, "sd_*_host: bad argument", cudaSuccess);
  if (n == 0) return SD_OK;
  DeviceGuard g(plan->device);
  const int64_t chunk = plan->chunk;
  const int64_t nchunks = (n + chunk - 1) / chunk;
  for (int64_t c = 0; c < nchunks; c++) {
    const int b = (int)(c % kBuf);
    cudaStream_t s = plan->stream[b];
    const int64_t r0 = c * chunk;
    const int64_t m = (n - r0) < chunk ? (n - r0) : chunk;
    Tin* din = static_cast<Tin*>(plan->in[b]);
    Tout* d0 = static_cast<Tout*>(plan->lam[b]);
    Tout* d1 = static_cast<Tout*>(plan->ang[b]);
    cudaError_t e = cudaMemcpyAsync(din, A + r0 * win, (size_t)m * win * sizeof(Tin),
                                    cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return herr(SD_ECUDA, "H2D copy", e);
    int rc = launch(din, m, d0, d1, plan->st[b], s);
    if (rc != SD_OK) return rc;  // sd_last_error() already set by the launcher
    e = cudaMemcpyAsync(out0 + r0 * w0, d0, (size_t)m * w0 * sizeof(Tout),
                        cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(out1 + r0 * w1, d1, (size_t)m * w1 * sizeof(Tout),
                          cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(status + r0, plan->st[b], (size_t)m, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return herr(SD_ECUDA, "D2H copy", e);
  }
  for (int b = 0; b < kBuf; b++) {
    cudaError_t e = cudaStreamSynchronize(plan->stream[b]);
    if (e != cudaSuccess) return herr(SD_ECUDA, "stream sync", e);
  }
  return SD_OK;
}

}  // namespace

extern "C" {

int sd_plan_create(int device, int64_t chunk, sd_plan** out) {
  if (!out || chunk <= 0) return herr(SD_EINVAL, "sd_plan_create: bad argument", cudaSuccess);
  *out = nullptr;
  sd_plan* p = new (std::nothrow) sd_plan;
  if (!p) return herr(SD_ENOMEM, "sd_plan_create: host allocation", cudaSuccess);
  p->device = device;
  p->chunk = chunk;
  DeviceGuard g(device);
  for (int b = 0; b < kBuf; b++) {
    cudaError_t e = cudaStreamCreateWithFlags(&p->stream[b], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&p->in[b], (size_t)chunk * 6 * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&p->lam[b], (size_t)chunk * 3 * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&p->ang[b], (size_t)chunk * 3 * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc((void**)&p->st[b], (size_t)chunk);
    if (e != cudaSuccess) {
      sd_plan_destroy(p);
      return herr(SD_ECUDA, "sd_plan_create", e);
    }
  }
  *out = p;
  return SD_OK;
}

int sd_plan_destroy(sd_plan* p) {
  if (!p) return SD_OK;
  DeviceGuard g(p->device);
  for (int b = 0; b < kBuf; b++) {
    if (p->stream[b]) cudaStreamSynchronize(p->stream[b]);
    cudaFree(p->in[b]);
    cudaFree(p->lam[b]);
    cudaFree(p->ang[b]);
    cudaFree(p->st[b]);
    if (p->stream[b]) cudaStreamDestroy(p->stream[b]);
  }
  delete p;
  return SD_OK;
}

int sd_eig3_f64_host(sd_plan* plan, const double* A, int64_t n, double* lam, double* ang,
                     uint8_t* status) {
  return run_pipeline<double, double>(
      plan, A, n, 6, lam, 3, ang, 3, status,
      [](const double* a, int64_t m, double* l, double* g, uint8_t* st, cudaStream_t s) {
        return sd_eig3_f64(a, m, l, g, st, s);
      });
}

int sd_eig3_f32_host(sd_plan* plan, const float* A, int64_t n, float* lam, float* ang,
                     uint8_t* status) {
  return run_pipeline<float, float>(
      plan, A, n, 6, lam, 3, ang, 3, status,
      [](const float* a, int64_t m, float* l, float* g, uint8_t* st, cudaStream_t s) {
        return sd_eig3_f32(a, m, l, g, st, s);
      });
}

int sd_eig2_f64_host(sd_plan* plan, const double* A, int64_t n, double* lam, double* phi,
                     uint8_t* status) {
  return run_pipeline<double, double>(
      plan, A, n, 3, lam, 2, phi, 1, status,
      [](const double* a, int64_t m, double* l, double* ph, uint8_t* st, cudaStream_t s) {
        return sd_eig2_f64(a, m, l, ph, st, s);
      });
}

}  // extern "C"
