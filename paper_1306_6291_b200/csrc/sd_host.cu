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
#include <cstring>
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
  double* rep = nullptr;   // chunk * SD_REPORT_STRIDE, allocated on first report call
  double* dmat = nullptr;  // chunk * 9
  // small synchronous calls: one packed device region and its pinned mirror,
  // so a call is one H2D copy, one launch and one D2H copy
  char* small_dev = nullptr;
  char* small_host = nullptr;
};

namespace {
constexpr int64_t kSmallRows = 64;
// per-row bytes of the packed small-call region: in 6 | lam 3 | ang 3 | rep 24 | d 9 doubles, st 1
constexpr int64_t kSmallBytes = kSmallRows * (6 + 3 + 3 + SD_REPORT_STRIDE + 9) * 8 + kSmallRows;
}  // namespace

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
  // on any error, wait for every stream before returning: copies already
  // queued into the caller's (possibly pinned) host buffers must not still
  // be running when the caller sees the error and frees or reuses them; the
  // first error code (and sd_last_error) is kept
  auto drain = [&](int rc) {
    for (int b = 0; b < kBuf; b++) cudaStreamSynchronize(plan->stream[b]);
    return rc;
  };
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
    if (e != cudaSuccess) return drain(herr(SD_ECUDA, "H2D copy", e));
    int rc = launch(din, m, d0, d1, plan->st[b], s);
    if (rc != SD_OK) return drain(rc);  // sd_last_error() already set by the launcher
    e = cudaMemcpyAsync(out0 + r0 * w0, d0, (size_t)m * w0 * sizeof(Tout),
                        cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(out1 + r0 * w1, d1, (size_t)m * w1 * sizeof(Tout),
                          cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(status + r0, plan->st[b], (size_t)m, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return drain(herr(SD_ECUDA, "D2H copy", e));
  }
  int rc = SD_OK;
  for (int b = 0; b < kBuf; b++) {
    cudaError_t e = cudaStreamSynchronize(plan->stream[b]);
    if (e != cudaSuccess && rc == SD_OK) rc = herr(SD_ECUDA, "stream sync", e);
  }
  return rc;
}

}  // namespace

namespace {
int ensure_report_buffers(sd_plan* p) {
  if (p->rep && p->dmat) return SD_OK;
  cudaError_t e = cudaMalloc(&p->rep, (size_t)p->chunk * SD_REPORT_STRIDE * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&p->dmat, (size_t)p->chunk * 9 * sizeof(double));
  return e == cudaSuccess ? SD_OK : herr(SD_ECUDA, "sd_*_report_host: allocation", e);
}

int ensure_small(sd_plan* p) {
  if (p->small_dev && p->small_host) return SD_OK;
  cudaError_t e = cudaMalloc((void**)&p->small_dev, kSmallBytes);
  if (e == cudaSuccess) e = cudaHostAlloc((void**)&p->small_host, kSmallBytes, cudaHostAllocMapped);
  return e == cudaSuccess ? SD_OK : herr(SD_ECUDA, "sd_*_report_host: allocation", e);
}

// Scalar-sized calls run zero-copy: the kernel reads A from, and writes
// every output to, the pinned mirror through its device mapping (a few
// hundred bytes over PCIe), so the call is one launch and one wait instead
// of H2D + launch + D2H (SD_SMALL_ZERO_COPY=0: the staged copies).
#ifndef SD_SMALL_ZERO_COPY
#define SD_SMALL_ZERO_COPY 1
#endif

// n <= kSmallRows: stage A in the pinned mirror, one H2D, `launch` on the
// packed device region, one D2H of every output, wait, unpack.
// Offsets (doubles): in 0, lam 6m, ang 9m, rep 12m, d 36m; status bytes at 45m.
template <typename Launch, typename Unpack>
int run_small(sd_plan* plan, int64_t m, int win, const double* A, Launch launch,
              Unpack unpack) {
  DeviceGuard g(plan->device);
  int rc = ensure_small(plan);
  if (rc != SD_OK) return rc;
  cudaStream_t s = plan->stream[0];
  double* h = reinterpret_cast<double*>(plan->small_host);
  double* dv = reinterpret_cast<double*>(plan->small_dev);
  std::memcpy(h, A, (size_t)m * win * sizeof(double));
  cudaError_t e;
#if SD_SMALL_ZERO_COPY
  double* hm = nullptr;  // device address of the mapped mirror
  if (cudaHostGetDevicePointer((void**)&hm, h, 0) == cudaSuccess && hm) {
    rc = launch(hm, hm + 6 * m, hm + 9 * m, hm + 12 * m, hm + 36 * m,
                reinterpret_cast<uint8_t*>(hm + 45 * m), s);
    if (rc != SD_OK) return rc;
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return herr(SD_ECUDA, "sd_*_report_host", e);
    unpack(h + 6 * m, h + 9 * m, h + 12 * m, h + 36 * m, reinterpret_cast<uint8_t*>(h + 45 * m));
    return SD_OK;
  }
  (void)cudaGetLastError();
#endif
  e = cudaMemcpyAsync(dv, h, (size_t)m * win * sizeof(double), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return herr(SD_ECUDA, "H2D copy", e);
  rc = launch(dv, dv + 6 * m, dv + 9 * m, dv + 12 * m, dv + 36 * m,
              reinterpret_cast<uint8_t*>(dv + 45 * m), s);
  if (rc != SD_OK) return rc;
  const size_t out_bytes = (size_t)m * 39 * sizeof(double) + (size_t)m;
  e = cudaMemcpyAsync(h + 6 * m, dv + 6 * m, out_bytes, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return herr(SD_ECUDA, "sd_*_report_host", e);
  unpack(h + 6 * m, h + 9 * m, h + 12 * m, h + 36 * m, reinterpret_cast<uint8_t*>(h + 45 * m));
  return SD_OK;
}

template <typename Launch, typename Copy>
int run_sync(sd_plan* plan, int64_t n, Launch launch, Copy copy_out) {
  DeviceGuard g(plan->device);
  int rc = ensure_report_buffers(plan);
  if (rc != SD_OK) return rc;
  cudaStream_t s = plan->stream[0];
  for (int64_t r0 = 0; r0 < n; r0 += plan->chunk) {
    const int64_t m = (n - r0) < plan->chunk ? (n - r0) : plan->chunk;
    rc = launch(r0, m, s);
    if (rc != SD_OK) return rc;
    cudaError_t e = copy_out(r0, m, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // host buffers may be pageable
    if (e != cudaSuccess) return herr(SD_ECUDA, "sd_*_report_host", e);
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
  cudaFree(p->rep);
  cudaFree(p->dmat);
  cudaFree(p->small_dev);
  if (p->small_host) cudaFreeHost(p->small_host);
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

// Synchronous host-buffer variants of the report entry points, for small
// batches and the reference-style scalar calls (one C call: copy in, one
// launch, copy out, wait).  Chunks of plan->chunk rows on the plan's first
// stream; no pipelining (latency, not throughput, is what these serve).

int sd_eig3_report_f64_host(sd_plan* plan, const double* A, int64_t n, double* lam, double* ang,
                            uint8_t* status, double* report, double* d) {
  if (!plan || n < 0 || (n > 0 && (!A || !lam || !ang || !status)))
    return herr(SD_EINVAL, "sd_eig3_report_f64_host: bad argument", cudaSuccess);
  if (n == 0) return SD_OK;
  if (n <= kSmallRows)
    return run_small(
        plan, n, 6, A,
        [&](double* din, double* dl, double* da, double* dr, double* dd, uint8_t* ds,
            cudaStream_t s) { return sd_eig3_report_f64(din, n, dl, da, ds, dr, dd, s); },
        [&](const double* hl, const double* ha, const double* hr, const double* hd,
            const uint8_t* hs) {
          std::memcpy(lam, hl, (size_t)n * 3 * sizeof(double));
          std::memcpy(ang, ha, (size_t)n * 3 * sizeof(double));
          std::memcpy(status, hs, (size_t)n);
          if (report) std::memcpy(report, hr, (size_t)n * SD_REPORT_STRIDE * sizeof(double));
          if (d) std::memcpy(d, hd, (size_t)n * 9 * sizeof(double));
        });
  double* din = static_cast<double*>(plan->in[0]);
  double* dl = static_cast<double*>(plan->lam[0]);
  double* da = static_cast<double*>(plan->ang[0]);
  return run_sync(
      plan, n,
      [&](int64_t r0, int64_t m, cudaStream_t s) {
        cudaError_t e = cudaMemcpyAsync(din, A + 6 * r0, (size_t)m * 6 * sizeof(double),
                                        cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return herr(SD_ECUDA, "H2D copy", e);
        return sd_eig3_report_f64(din, m, dl, da, plan->st[0], report ? plan->rep : nullptr,
                                  d ? plan->dmat : nullptr, s);
      },
      [&](int64_t r0, int64_t m, cudaStream_t s) {
        cudaError_t e = cudaMemcpyAsync(lam + 3 * r0, dl, (size_t)m * 3 * sizeof(double),
                                        cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(ang + 3 * r0, da, (size_t)m * 3 * sizeof(double),
                              cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(status + r0, plan->st[0], (size_t)m, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess && report)
          e = cudaMemcpyAsync(report + SD_REPORT_STRIDE * r0, plan->rep,
                              (size_t)m * SD_REPORT_STRIDE * sizeof(double),
                              cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess && d)
          e = cudaMemcpyAsync(d + 9 * r0, plan->dmat, (size_t)m * 9 * sizeof(double),
                              cudaMemcpyDeviceToHost, s);
        return e;
      });
}

int sd_eig2_report_f64_host(sd_plan* plan, const double* A, int64_t n, double* lam, double* phi,
                            uint8_t* status, double* d) {
  if (!plan || n < 0 || (n > 0 && (!A || !lam || !phi || !status)))
    return herr(SD_EINVAL, "sd_eig2_report_f64_host: bad argument", cudaSuccess);
  if (n == 0) return SD_OK;
  if (n <= kSmallRows)
    return run_small(
        plan, n, 3, A,
        [&](double* din, double* dl, double* dp, double*, double* dd, uint8_t* ds,
            cudaStream_t s) { return sd_eig2_report_f64(din, n, dl, dp, ds, dd, s); },
        [&](const double* hl, const double* hp, const double*, const double* hd,
            const uint8_t* hs) {
          std::memcpy(lam, hl, (size_t)n * 2 * sizeof(double));
          std::memcpy(phi, hp, (size_t)n * sizeof(double));
          std::memcpy(status, hs, (size_t)n);
          if (d) std::memcpy(d, hd, (size_t)n * 4 * sizeof(double));
        });
  double* din = static_cast<double*>(plan->in[0]);
  double* dl = static_cast<double*>(plan->lam[0]);
  double* dp = static_cast<double*>(plan->ang[0]);
  return run_sync(
      plan, n,
      [&](int64_t r0, int64_t m, cudaStream_t s) {
        cudaError_t e = cudaMemcpyAsync(din, A + 3 * r0, (size_t)m * 3 * sizeof(double),
                                        cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return herr(SD_ECUDA, "H2D copy", e);
        return sd_eig2_report_f64(din, m, dl, dp, plan->st[0], d ? plan->dmat : nullptr, s);
      },
      [&](int64_t r0, int64_t m, cudaStream_t s) {
        cudaError_t e = cudaMemcpyAsync(lam + 2 * r0, dl, (size_t)m * 2 * sizeof(double),
                                        cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(phi + r0, dp, (size_t)m * sizeof(double), cudaMemcpyDeviceToHost,
                              s);
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(status + r0, plan->st[0], (size_t)m, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess && d)
          e = cudaMemcpyAsync(d + 4 * r0, plan->dmat, (size_t)m * 4 * sizeof(double),
                              cudaMemcpyDeviceToHost, s);
        return e;
      });
}

}  // extern "C"
