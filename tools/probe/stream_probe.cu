// Streaming probe: TMA box loads over a column-major f64 matrix with the SJLT
// kernel's tile order, no compute -- the HBM ceiling of the access pattern.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//        -I../../paper_2302_01977_b200/csrc -I../../include stream_probe.cu ../../paper_2302_01977_b200/csrc/hsk_misc.cu -lcuda -o stream_probe.so
#include "hsk_common.cuh"

using namespace hsk;

struct PArgs {
    int64_t rows, cols;
    int box_r, box_c, stages, nslabs, tiles, nchunks, persistent;
    double *sink;
};

__global__ void __launch_bounds__(128, 1) probe_kernel(const PArgs p, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    unsigned char *st0 = smem + 1024;
    const uint32_t bytes = p.box_r * p.box_c * 8;
    int64_t u0, u1;
    if (p.persistent) {
        const int64_t groups = gridDim.x / p.nslabs, grp = blockIdx.x / p.nslabs;
        const int64_t units = (int64_t)p.tiles * p.nchunks;
        u0 = grp * units / groups;
        u1 = (grp + 1) * units / groups;
    } else {
        const int64_t tile = blockIdx.x / p.nslabs;
        u0 = tile * p.nchunks;
        u1 = u0 + p.nchunks;
    }
    const int n = (int)(u1 - u0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    double acc = 0;
    if (threadIdx.x == 0) {
        auto issue = [&](int j) {
            const int64_t u = u0 + j, t = u / p.nchunks, c = u - t * p.nchunks;
            uint64_t *bar = &full[j % p.stages];
            mbar_arrive_expect_tx(bar, bytes);
            tma_load_2d(st0 + (size_t)(j % p.stages) * bytes, &tmap, (int)(t * p.box_r), (int)(c * p.box_c), bar);
        };
        for (int j = 0; j < n && j < p.stages; ++j) issue(j);
        for (int j = 0; j < n; ++j) {
            mbar_wait(&full[j % p.stages], (uint32_t)(j / p.stages) & 1u);
            acc += reinterpret_cast<double *>(st0 + (size_t)(j % p.stages) * bytes)[j & 63];
            if (j + p.stages < n) issue(j + p.stages);
        }
        p.sink[blockIdx.x] = acc;
    }
}

extern "C" int probe_run(const double *A, int64_t rows, int64_t cols, int box_r, int box_c, int stages,
                         int nslabs, int persistent, int grid_override, double *sink, void *stream) {
    CUtensorMap tmap;
    int rc = make_tmap_f64_2d(&tmap, A, rows, cols, rows, box_r, box_c);
    if (rc) return rc;
    PArgs p;
    p.rows = rows;
    p.cols = cols;
    p.box_r = box_r;
    p.box_c = box_c;
    p.stages = stages;
    p.nslabs = nslabs;
    p.tiles = (int)((rows + box_r - 1) / box_r);
    p.nchunks = (int)((cols + box_c - 1) / box_c);
    p.persistent = persistent;
    p.sink = sink;
    const int smem = 1024 + stages * box_r * box_c * 8;
    cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int grid = persistent ? (grid_override > 0 ? grid_override : sm_count() / nslabs * nslabs) : p.tiles * nslabs;
    probe_kernel<<<grid, 128, smem, (cudaStream_t)stream>>>(p, tmap);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}
