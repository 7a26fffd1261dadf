// Host<->device copy bandwidth: 1-D cudaMemcpyAsync vs the engine's pitched
// cudaMemcpy2DAsync, pinned host memory, 4100 x 4100 doubles (one padded
// field of the bench grid) per copy.
#include <cstdio>
#include <cuda_runtime.h>

int main() {
    const size_t rows = 4100, cols = 4100, dpitch = 4128;
    const size_t bytes = rows * cols * 8;
    double *h, *d, *d2;
    cudaMallocHost(&h, bytes);
    cudaMalloc(&d, rows * dpitch * 8);
    cudaMalloc(&d2, bytes);
    for (size_t i = 0; i < rows * cols; i++) h[i] = double(i);
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char *name, auto fn) {
        fn();
        cudaStreamSynchronize(st);
        cudaEventRecord(a, st);
        for (int k = 0; k < 5; k++) fn();
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-28s %.1f GB/s\n", name, 5.0 * bytes / (ms * 1e-3) / 1e9);
    };
    run("H2D 1-D", [&] { cudaMemcpyAsync(d2, h, bytes, cudaMemcpyHostToDevice, st); });
    run("H2D 2-D pitched", [&] {
        cudaMemcpy2DAsync(d + 28, dpitch * 8, h, cols * 8, cols * 8, rows, cudaMemcpyHostToDevice, st);
    });
    run("D2H 1-D", [&] { cudaMemcpyAsync(h, d2, bytes, cudaMemcpyDeviceToHost, st); });
    run("D2H 2-D pitched", [&] {
        cudaMemcpy2DAsync(h, cols * 8, d + 28, dpitch * 8, cols * 8, rows, cudaMemcpyDeviceToHost, st);
    });
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
