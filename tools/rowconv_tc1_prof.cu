// Wait-time breakdown of the tcgen05 row operator (rowconv_tc1) per warp role.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTIDAS_RC_PROF \
//        -o build/var/rowconv_tc1_prof tools/rowconv_tc1_prof.cu paper_2507_15464_b200/csrc/api.cu -lcuda
//   build/var/rowconv_tc1_prof [batch nz nx]      (default: cfg2 maps 512 x 512 x 256)
#include "../paper_2507_15464_b200/csrc/rowconv_tc1.cu"
#include <cstdio>
#include <cstdlib>
#include <cstring>

int main(int argc, char** argv) {
  const int B = argc > 3 ? atoi(argv[1]) : 512, nz = argc > 3 ? atoi(argv[2]) : 512, nx = argc > 3 ? atoi(argv[3]) : 256;
  const int T = 129;
  float *in, *K, *out;
  cudaMalloc(&in, (size_t)B * nz * nx * 4);
  cudaMalloc(&out, (size_t)B * nz * nx * 4);
  cudaMalloc(&K, (size_t)nz * T * 4);
  cudaMemset(in, 0, (size_t)B * nz * nx * 4);
  cudaMemset(K, 0, (size_t)nz * T * 4);
  for (int i = 0; i < 3; ++i) tidas::launch_rowconv_tc1<false>(in, K, out, B, nz, nx, T, 0);
  cudaDeviceSynchronize();
  unsigned long long z[16][16];
  memset(z, 0, sizeof(z));
  cudaMemcpyToSymbol(tidas::tcx::g_rc_prof, z, sizeof(z));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int rc = tidas::launch_rowconv_tc1<false>(in, K, out, B, nz, nx, T, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaMemcpyFromSymbol(z, tidas::tcx::g_rc_prof, sizeof(z));
  const double gbs = 2.0 * B * nz * nx * 4 / (ms * 1e-3) / 1e9;
  printf("B=%d nz=%d nx=%d rc=%d  %.4f ms  %.0f GB/s (%s)\n", B, nz, nx, rc, ms, gbs, cudaGetErrorString(cudaGetLastError()));
  const char* site[10] = {"row_done", "c_free", "a_full", "mma_done", "a_empty", "c_full", "d_empty", "b_full", "issue", "TOTAL"};
  const char* role[16] = {"conv0", "conv1", "conv2", "conv3", "epi0", "epi1", "epi2", "epi3", "mma", "tma",
                          "bld0", "bld1", "conv4", "conv5", "conv6", "conv7"};
  for (int w = 0; w < 16; ++w) {
    printf("%-6s", role[w]);
    const double tot = (double)z[w][9];
    for (int k = 0; k < 9; ++k)
      if (z[w][k]) printf("  %s %4.1f%%", site[k], 100.0 * z[w][k] / tot);
    printf("  | total %.0f cyc/CTA\n", tot / 148);
  }
  return 0;
}
