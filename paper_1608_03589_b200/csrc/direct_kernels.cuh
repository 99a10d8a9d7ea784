// Direct pixel-driven backprojector (reference.py:21-37): geometry and launcher.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace lpbp {

struct DirectGeom {
  int nt, ntheta, n;
  int pad, ntp;      // zero entries on each side of a packed angle row; row length nt + 2 pad
  int groups;        // slice groups of 4 (the last one zero-padded)
  int W, A;          // window entries per angle and angles per shared-memory stage
  size_t tab_bytes;  // angle table (float2 [ntheta]) at the workspace start, 256-byte padded
  size_t ws_bytes;   // angle table + packed rows float4 [groups][ntheta][ntp]
  size_t smem;       // dynamic shared memory of k_direct
};

int direct_pad(int nt);
DirectGeom direct_geom(int nt, int ntheta, int n, int batch);
// sino [batch][nt][ntheta] -> img [batch][n][n]; ws: g.ws_bytes, 256-byte aligned. Two launches.
cudaError_t launch_direct(const DirectGeom& g, const float* sino, void* ws, float* img, int batch, cudaStream_t s);

}  // namespace lpbp
