// Probe: stream memory operations through the runtime's driver entry points.
#include <cuda_runtime.h>
#include <cstdio>
typedef int (*Fn)(cudaStream_t, unsigned long long, unsigned int, unsigned int);
int main() {
    cudaSetDevice(0);
    cudaFree(0);
    void *w = nullptr, *v = nullptr;
    cudaDriverEntryPointQueryResult q1, q2;
    cudaError_t e1 = cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &q1);
    cudaError_t e2 = cudaGetDriverEntryPoint("cuStreamWaitValue32", &v, cudaEnableDefault, &q2);
    printf("entry: %s %d %p | %s %d %p\n", cudaGetErrorName(e1), (int)q1, w, cudaGetErrorName(e2), (int)q2, v);
    void* w2 = nullptr; cudaDriverEntryPointQueryResult q3;
    cudaError_t e3 = cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &w2, 12000, cudaEnableDefault, &q3);
    printf("byversion: %s %d %p\n", cudaGetErrorName(e3), (int)q3, w2);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    unsigned* d;
    cudaMalloc(&d, 64);
    cudaMemset(d, 0, 64);
    int r = ((Fn)w)(s, (unsigned long long)d, 7u, 0u);
    printf("write rc=%d\n", r);
    r = ((Fn)v)(s, (unsigned long long)d, 7u, 0u);
    printf("wait rc=%d\n", r);
    cudaStreamSynchronize(s);
    unsigned h = 0;
    cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("value=%u err=%s\n", h, cudaGetErrorName(cudaGetLastError()));
    if (w2) { r = ((Fn)w2)(s, (unsigned long long)(d + 1), 9u, 0u); cudaStreamSynchronize(s);
      cudaMemcpy(&h, d + 1, 4, cudaMemcpyDeviceToHost); printf("v2 write rc=%d value=%u\n", r, h); }
    return 0;
}
