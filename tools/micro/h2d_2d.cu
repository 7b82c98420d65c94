// H2D bandwidth of column-slab uploads: a 65536 x 8 KB pinned host matrix copied as
// one contiguous block vs as W-byte-wide column slabs (cudaMemcpy2DAsync), to size the
// e2e upload pipeline.  nvcc -O2 -o h2d_2d h2d_2d.cu
#include <cstdio>
#include <cuda_runtime.h>
int main() {
    const size_t rows = 65536, pitch = 8192 + 128, row = 8192;
    char *h, *d;
    cudaHostAlloc(&h, rows * row, cudaHostAllocDefault);
    cudaMalloc(&d, rows * pitch);
    for (size_t i = 0; i < rows * row; i += 4096) h[i] = 1;
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep)
        for (size_t w : {size_t(8192), size_t(4096), size_t(2048), size_t(1024), size_t(512), size_t(128)}) {
            cudaEventRecord(a, s);
            for (size_t c = 0; c < row; c += w)
                cudaMemcpy2DAsync(d + c, pitch, h + c, row, w, rows, cudaMemcpyHostToDevice, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("slab %5zu B: %.3f ms  %.1f GB/s\n", w, ms, rows * row / ms / 1e6);
        }
    return 0;
}
