#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
struct S { cudaStream_t ci = nullptr, kk = nullptr, co = nullptr; cudaEvent_t a = nullptr, b = nullptr, c = nullptr, d = nullptr, e = nullptr; };
int main(int argc, char**) {
    cudaSetDevice(0);
    cudaFree(0);
    void *w = nullptr; cudaDriverEntryPointQueryResult q1;
    if (argc > 1) cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &q1);
    S s;
    cudaStreamCreateWithFlags(&s.ci, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s.kk, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s.co, cudaStreamNonBlocking);
    for (cudaEvent_t* e : {&s.a, &s.b, &s.c, &s.d, &s.e}) { cudaError_t r = cudaEventCreate(e); printf("create %s %p\n", cudaGetErrorName(r), (void*)*e); }
    cudaError_t r = cudaEventRecord(s.a, s.ci);
    printf("record %s\n", cudaGetErrorName(r));
    return 0;
}
