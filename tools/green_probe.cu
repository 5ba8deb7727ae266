// Probe: SM partitioning with green contexts (driver API via cudaGetDriverEntryPoint,
// no libcuda link). Checks that runtime launches into green-context streams run on the
// partition's SMs, see memory from cudaMalloc, order against primary-context streams
// by events, and that a graph captured in a green stream replays there.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <set>
#include <vector>

#define CK(x) do { auto e_ = (x); if (e_ != 0) { std::printf("FAIL %s = %d (line %d)\n", #x, (int)e_, __LINE__); return 1; } } while (0)

__global__ void smid_kernel(int* out, int n)
{
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = s;
}
__global__ void spin_kernel(double* x, int n, int reps)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double v = x[i];
    for (int r = 0; r < reps; ++r) v = v * 0.999999 + 1e-9;
    x[i] = v;
  }
}

template <class F>
F sym(const char* name)
{
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPointByVersion(name, &p, 12090, cudaEnableDefault, &q) != cudaSuccess || !p) {
    std::printf("no symbol %s\n", name);
    return nullptr;
  }
  return reinterpret_cast<F>(p);
}

int main()
{
  CK(cudaSetDevice(0));
  CK(cudaFree(0));
  auto pGetRes = sym<CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType)>("cuDeviceGetDevResource");
  auto pSplit = sym<CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned)>(
      "cuDevSmResourceSplitByCount");
  auto pDesc = sym<CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned)>("cuDevResourceGenerateDesc");
  auto pCreate = sym<CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned)>("cuGreenCtxCreate");
  auto pStream = sym<CUresult (*)(CUstream*, CUgreenCtx, unsigned, int)>("cuGreenCtxStreamCreate");
  auto pFromGreen = sym<CUresult (*)(CUcontext*, CUgreenCtx)>("cuCtxFromGreenCtx");
  auto pSetCur = sym<CUresult (*)(CUcontext)>("cuCtxSetCurrent");
  auto pGetCur = sym<CUresult (*)(CUcontext*)>("cuCtxGetCurrent");
  if (!pGetRes || !pSplit || !pDesc || !pCreate || !pStream || !pFromGreen || !pSetCur || !pGetCur) return 1;
  CUdevResource all{};
  CK(pGetRes(0, &all, CU_DEV_RESOURCE_TYPE_SM));
  std::printf("device SMs %u\n", all.sm.smCount);
  for (unsigned want : {8u, 16u, 24u}) {
    CUdevResource part{}, rest{};
    unsigned nb = 1;
    CK(pSplit(&part, &nb, &all, &rest, 0, want));
    std::printf("split %u -> groups %u part %u rest %u\n", want, nb, part.sm.smCount, rest.sm.smCount);
  }
  CUdevResource part{}, rest{};
  unsigned nb = 1;
  CK(pSplit(&part, &nb, &all, &rest, 0, 16));
  CUdevResourceDesc dA, dB;
  CK(pDesc(&dA, &part, 1));
  CK(pDesc(&dB, &rest, 1));
  CUgreenCtx gA, gB;
  CK(pCreate(&gA, dA, 0, CU_GREEN_CTX_DEFAULT_STREAM));
  CK(pCreate(&gB, dB, 0, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sA, sB;
  CK(pStream(&sA, gA, CU_STREAM_NON_BLOCKING, -1));
  CK(pStream(&sB, gB, CU_STREAM_NON_BLOCKING, 0));
  CUcontext prim, cA, cB;
  CK(pGetCur(&prim));
  CK(pFromGreen(&cA, gA));
  CK(pFromGreen(&cB, gB));
  const int n = 1 << 20;
  int* d_sm;
  CK(cudaMalloc(&d_sm, n * sizeof(int)));  // primary-context allocation
  std::vector<int> h(n);
  // 1: launch into sA with the primary context current
  smid_kernel<<<1184, 256, 0, (cudaStream_t)sA>>>(d_sm, n);
  std::printf("launch (primary current) into green stream: %s\n", cudaGetErrorString(cudaGetLastError()));
  CK(cudaStreamSynchronize((cudaStream_t)sA));
  CK(cudaMemcpy(h.data(), d_sm, n * sizeof(int), cudaMemcpyDeviceToHost));
  std::set<int> sa(h.begin(), h.end());
  std::printf("stream A ran on %zu SMs (min %d max %d)\n", sa.size(), *sa.begin(), *sa.rbegin());
  smid_kernel<<<1184, 256, 0, (cudaStream_t)sB>>>(d_sm, n);
  CK(cudaStreamSynchronize((cudaStream_t)sB));
  CK(cudaMemcpy(h.data(), d_sm, n * sizeof(int), cudaMemcpyDeviceToHost));
  std::set<int> sb(h.begin(), h.end());
  int overlap = 0;
  for (int x : sb) overlap += sa.count(x);
  std::printf("stream B ran on %zu SMs, overlap with A: %d\n", sb.size(), overlap);
  // 2: events between a primary stream and green streams
  cudaStream_t sp;
  CK(cudaStreamCreateWithFlags(&sp, cudaStreamNonBlocking));
  cudaEvent_t e0, e1, e2, t0, t1;
  CK(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
  CK(cudaEventCreate(&t0));
  CK(cudaEventCreate(&t1));
  double* x;
  const int m = 148 * 2048 * 4;
  CK(cudaMalloc(&x, m * sizeof(double)));
  CK(cudaMemset(x, 0, m * sizeof(double)));
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaEventRecord(t0, sp));
    CK(cudaEventRecord(e0, sp));
    CK(cudaStreamWaitEvent((cudaStream_t)sA, e0, 0));
    CK(cudaStreamWaitEvent((cudaStream_t)sB, e0, 0));
    spin_kernel<<<148 * 8, 256, 0, (cudaStream_t)sA>>>(x, m / 2, 2000);
    spin_kernel<<<148 * 8, 256, 0, (cudaStream_t)sB>>>(x + m / 2, m / 2, 2000);
    CK(cudaEventRecord(e1, (cudaStream_t)sA));
    CK(cudaEventRecord(e2, (cudaStream_t)sB));
    CK(cudaStreamWaitEvent(sp, e1, 0));
    CK(cudaStreamWaitEvent(sp, e2, 0));
    CK(cudaEventRecord(t1, sp));
    CK(cudaEventSynchronize(t1));
    float ms;
    CK(cudaEventElapsedTime(&ms, t0, t1));
    std::printf("fork/join over green streams: %.3f ms (%s)\n", ms, cudaGetErrorString(cudaGetLastError()));
  }
  // 3: graph captured in a green stream, replayed there
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture((cudaStream_t)sA, cudaStreamCaptureModeThreadLocal));
  for (int k = 0; k < 10; ++k) smid_kernel<<<64, 256, 0, (cudaStream_t)sA>>>(d_sm, n);
  CK(cudaStreamEndCapture((cudaStream_t)sA, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, (cudaStream_t)sA));
  CK(cudaStreamSynchronize((cudaStream_t)sA));
  CK(cudaMemcpy(h.data(), d_sm, n * sizeof(int), cudaMemcpyDeviceToHost));
  std::set<int> sg(h.begin(), h.end());
  int ov = 0;
  for (int v : sg) ov += sa.count(v);
  std::printf("graph captured in A replayed: %zu SMs, all in A: %s\n", sg.size(), ov == (int)sg.size() ? "yes" : "no");
  // graph captured in a primary stream launched into A
  CK(cudaStreamBeginCapture(sp, cudaStreamCaptureModeThreadLocal));
  for (int k = 0; k < 10; ++k) smid_kernel<<<64, 256, 0, sp>>>(d_sm, n);
  CK(cudaStreamEndCapture(sp, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  cudaError_t le = cudaGraphLaunch(ge, (cudaStream_t)sA);
  std::printf("primary-captured graph launched into A: %s\n", cudaGetErrorString(le));
  CK(cudaStreamSynchronize((cudaStream_t)sA));
  CK(cudaMemcpy(h.data(), d_sm, n * sizeof(int), cudaMemcpyDeviceToHost));
  std::set<int> sg2(h.begin(), h.end());
  ov = 0;
  for (int v : sg2) ov += sa.count(v);
  std::printf("  ran on %zu SMs, all in A: %s\n", sg2.size(), ov == (int)sg2.size() ? "yes" : "no");
  std::printf("OK\n");
  return 0;
}
