// datagen.cu -- seeded synthetic inputs shaped like the paper's workloads (device side).
//
// Shared by tests, bench.py and the product demo; holds none of the method's arithmetic.
// Random-walk series (sec. 5 "Datasets": "a random number is first drawn from
// a Gaussian distribution N(0,1), and then at each time point a new number is drawn from
// this distribution and added to the value of the last number"), z-normalised.
// Counter-based generator: Philox4x32-10 keyed by the seed, counter = (pair index, row,
// stream), Box-Muller in fp64, cumulative sum and population z-normalisation in fp64,
// one rounding to fp32.  datagen/__init__.py holds the same generator in numpy.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr uint32_t kStreamWalk = 0, kStreamRows = 1, kStreamNoise = 2;

struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                     uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return {c0, c1, c2, c3};
}

// Standard normal pair j (numbers 2j, 2j+1) of (seed, row, stream): Box-Muller on one
// Philox block.
__device__ __forceinline__ void normal_pair(uint64_t seed, uint64_t row, uint32_t stream, int j,
                                            double& z0, double& z1)
{
    U4 r = philox((uint32_t)j, (uint32_t)row, (uint32_t)(row >> 32), stream, (uint32_t)seed,
                  (uint32_t)(seed >> 32));
    uint64_t a = ((uint64_t)r.y << 32) | r.x, b = ((uint64_t)r.w << 32) | r.z;
    double u1 = (double)((a >> 11) + 1) * 0x1.0p-53;  // (0, 1]
    double u2 = (double)(b >> 11) * 0x1.0p-53;        // [0, 1)
    double rad = sqrt(-2.0 * log(u1));
    double ang = 6.283185307179586 * u2;
    z0 = rad * cos(ang);
    z1 = rad * sin(ang);
}

// z-normalised random walk of (seed, row), written as fp32 into out[0..n) (n even).  Three
// passes (mean, population variance, write) regenerate the walk instead of holding n doubles.
__device__ void walk_row(uint64_t seed, uint64_t row, int n, float* out)
{
    double x = 0.0, sum = 0.0, z0, z1;
    for (int j = 0; j < n / 2; ++j) {
        normal_pair(seed, row, kStreamWalk, j, z0, z1);
        x += z0; sum += x;
        x += z1; sum += x;
    }
    double mu = sum / n;
    double ss = 0.0;
    x = 0.0;
    for (int j = 0; j < n / 2; ++j) {
        normal_pair(seed, row, kStreamWalk, j, z0, z1);
        x += z0; ss += (x - mu) * (x - mu);
        x += z1; ss += (x - mu) * (x - mu);
    }
    double sd = sqrt(ss / n);
    x = 0.0;
    for (int j = 0; j < n / 2; ++j) {
        normal_pair(seed, row, kStreamWalk, j, z0, z1);
        x += z0; out[2 * j] = sd > 0.0 ? (float)((x - mu) / sd) : 0.0f;
        x += z1; out[2 * j + 1] = sd > 0.0 ? (float)((x - mu) / sd) : 0.0f;
    }
}

__global__ void walks_kernel(float* out, int64_t row_begin, int64_t rows, int n, uint64_t seed)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= rows) return;
    walk_row(seed, (uint64_t)(row_begin + k), n, out + k * (int64_t)n);
}

// Query qi of the noise workload (BASELINE config 5): a uniformly chosen
// dataset row plus N(0, sigma^2) per point, re-z-normalised.  out must hold n floats of
// scratch per query (it first receives the source row).
__global__ void noisy_kernel(float* out, int nq, int n, int64_t N, uint64_t data_seed,
                             uint64_t query_seed, double sigma)
{
    int qi = blockIdx.x * blockDim.x + threadIdx.x;
    if (qi >= nq) return;
    U4 r = philox(0u, (uint32_t)qi, 0u, kStreamRows, (uint32_t)query_seed, (uint32_t)(query_seed >> 32));
    uint64_t u = ((uint64_t)r.y << 32) | r.x;
    uint64_t row = __umul64hi(u, (uint64_t)N);
    float* q = out + (int64_t)qi * n;
    walk_row(data_seed, row, n, q);
    double z0, z1, sum = 0.0;
    for (int j = 0; j < n / 2; ++j) {
        normal_pair(query_seed, (uint64_t)qi, kStreamNoise, j, z0, z1);
        sum += (double)q[2 * j] + sigma * z0;
        sum += (double)q[2 * j + 1] + sigma * z1;
    }
    double mu = sum / n, ss = 0.0;
    for (int j = 0; j < n / 2; ++j) {
        normal_pair(query_seed, (uint64_t)qi, kStreamNoise, j, z0, z1);
        double v0 = (double)q[2 * j] + sigma * z0 - mu, v1 = (double)q[2 * j + 1] + sigma * z1 - mu;
        ss += v0 * v0;
        ss += v1 * v1;
    }
    double sd = sqrt(ss / n);
    for (int j = 0; j < n / 2; ++j) {
        normal_pair(query_seed, (uint64_t)qi, kStreamNoise, j, z0, z1);
        double v0 = (double)q[2 * j] + sigma * z0, v1 = (double)q[2 * j + 1] + sigma * z1;
        q[2 * j] = sd > 0.0 ? (float)((v0 - mu) / sd) : 0.0f;
        q[2 * j + 1] = sd > 0.0 ? (float)((v1 - mu) / sd) : 0.0f;
    }
}

}  // namespace

extern "C" {

// Rows [row_begin, row_begin+rows) of the z-normalised random-walk collection `seed`,
// row-major fp32 into device memory out[rows][n].  Returns 0 or a cudaError_t.
int dg_random_walks(float* out, int64_t row_begin, int64_t rows, int n, uint64_t seed, void* stream)
{
    if (rows <= 0) return 0;
    int threads = 128;
    int64_t blocks = (rows + threads - 1) / threads;
    walks_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(out, row_begin, rows, n, seed);
    return (int)cudaGetLastError();
}

// nq noisy queries (config 5) over a collection of N rows generated with data_seed.
int dg_noisy_queries(float* out, int nq, int n, int64_t N, uint64_t data_seed, uint64_t query_seed,
                     double sigma, void* stream)
{
    if (nq <= 0) return 0;
    int threads = 64;
    noisy_kernel<<<(nq + threads - 1) / threads, threads, 0, (cudaStream_t)stream>>>(
        out, nq, n, N, data_seed, query_seed, sigma);
    return (int)cudaGetLastError();
}

}  // extern "C"
