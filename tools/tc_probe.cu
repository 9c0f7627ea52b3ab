// Standalone launcher for the tcgen05 conv (prints the CUDA error string).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2306_17486_b200/csrc/conv_tc.h"

int main(int argc, char** argv) {
  int B = argc > 1 ? atoi(argv[1]) : 1, H = argc > 2 ? atoi(argv[2]) : 128, W = argc > 3 ? atoi(argv[3]) : 128;
  int cin = 16, cout = 16;
  size_t nx = (size_t)B * H * W * cin, ny = (size_t)B * H * W * cout;
  std::vector<float> hx(nx), hw(cout * 9 * cin), hb(cout, 0.1f);
  for (size_t i = 0; i < nx; ++i) hx[i] = (float)((i * 2654435761u) % 1000) / 1000.f - 0.5f;
  for (size_t i = 0; i < hw.size(); ++i) hw[i] = (float)((i * 40503u) % 100) / 100.f - 0.5f;
  float *x, *w, *b, *y;
  cudaMalloc(&x, nx * 4);
  cudaMalloc(&w, hw.size() * 4);
  cudaMalloc(&b, cout * 4);
  cudaMalloc(&y, ny * 4);
  cudaMemcpy(x, hx.data(), nx * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(w, hw.data(), hw.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(b, hb.data(), cout * 4, cudaMemcpyHostToDevice);
  printf("launching B=%d H=%d W=%d\n", B, H, W);
  fflush(stdout);
  hs::conv_tc_launch(x, H, W, cin, y, H, W, cout, 1, 0, w, b, 1, nullptr, 0, 0, nullptr, nullptr, nullptr, B, 0);
  printf("launch: %s\n", cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
  cudaError_t e = cudaDeviceSynchronize();
  printf("sync: %s\n", cudaGetErrorString(e));
  std::vector<float> hy(ny);
  cudaMemcpy(hy.data(), y, ny * 4, cudaMemcpyDeviceToHost);
  // reference for a few pixels
  double maxerr = 0;
  for (int t = 0; t < 200; ++t) {
    int bb = t % B, oy = (t * 37) % H, ox = (t * 91) % W, n = t % cout;
    double acc = hb[n];
    for (int ky = 0; ky < 3; ++ky)
      for (int kx = 0; kx < 3; ++kx) {
        int iy = oy + ky - 1, ix = ox + kx - 1;
        if (iy < 0 || iy >= H || ix < 0 || ix >= W) continue;
        for (int c = 0; c < cin; ++c)
          acc += (double)hx[(((size_t)bb * H + iy) * W + ix) * cin + c] * hw[((size_t)n * 9 + ky * 3 + kx) * cin + c];
      }
    double sp = acc > 0 ? acc + log1p(exp(-acc)) : log1p(exp(acc));
    double got = hy[(((size_t)bb * H + oy) * W + ox) * cout + n];
    double err = fabs(got - sp) / (fabs(sp) + 1e-6);
    if (err > maxerr) maxerr = err;
  }
  printf("max rel err %.3e\n", maxerr);
  return 0;
}
