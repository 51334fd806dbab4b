// bruteforce.cu — the reference's brute-force renderer (inc/oracle.hpp:161-270) on the GPU, in
// double: an independent validation path for large scenes, sharing no code
// with the fast pipeline (own projection transcription, own covariance, own SH table, a
// global (depth, source) order instead of tile lists, every splat gated per tile).
//
//   bf_splats_kernel  per Gaussian: oracle_project (oracle.hpp:103-158, incl. the fisheye axis
//                     limit), Sigma = R diag(s^2) R^T from the normalised quaternion, T = J W,
//                     Sigma_p + 0.3 I, det / radius / off-screen cull, conic, depth, colour
//                     (oracle_sh_color, :70-99), alpha = 1 / (1 + e^-x)           (:161-218)
//   [host: stable sort of the kept splats by (depth, source)]
//   bf_render_kernel  one CTA per 16x16 tile walks the whole sorted list in 256-splat chunks:
//                     the tile-overlap gate (:251-254) is evaluated cooperatively and the
//                     survivors are blended by every pixel in order, in double (:255-266).

#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "../../include/fgs.h"
#include "fgs_kernels.h"

namespace fgs {

namespace {

constexpr int kBfTile = 16;
constexpr double kBfPi = 3.141592653589793238462643383279502884;

struct BfSplat {
  double mx, my, ca, cb, cc, depth, r, g, b, alpha;
  int radius, source;
};

template <typename Real>
__device__ double bf_sh(const Real* c, const double d[3], int degree) {
  double v = 0.28209479177387814 * c[0];
  if (degree >= 1) v += -0.4886025119029199 * d[1] * c[1] + 0.4886025119029199 * d[2] * c[2] - 0.4886025119029199 * d[0] * c[3];
  if (degree >= 2) {
    const double xx = d[0] * d[0], yy = d[1] * d[1], zz = d[2] * d[2];
    v += 1.0925484305920792 * d[0] * d[1] * c[4] - 1.0925484305920792 * d[1] * d[2] * c[5] +
         0.31539156525252005 * (2.0 * zz - xx - yy) * c[6] - 1.0925484305920792 * d[0] * d[2] * c[7] +
         0.5462742152960396 * (xx - yy) * c[8];
  }
  if (degree >= 3) {
    const double x = d[0], y = d[1], z = d[2], xx = x * x, yy = y * y, zz = z * z;
    v += -0.5900435899266435 * y * (3.0 * xx - yy) * c[9] + 2.890611442640554 * x * y * z * c[10] -
         0.4570457994644658 * y * (4.0 * zz - xx - yy) * c[11] +
         0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy) * c[12] -
         0.4570457994644658 * x * (4.0 * zz - xx - yy) * c[13] + 1.445305721320277 * z * (xx - yy) * c[14] -
         0.5900435899266435 * x * (xx - yy) * c[15];
  }
  return fmax(v + 0.5, 0.0);
}

__device__ bool bf_project(const double p[3], const fgs_camera& cam, double pix[2], double j[2][3]) {
  const double x = p[0], y = p[1], z = p[2];
  if (x * x + y * y + z * z < 1e-24) return false;
  const double fx = cam.fx, fy = cam.fy, cx = cam.cx, cy = cam.cy;
  if (cam.model == FGS_CAMERA_PINHOLE || cam.model == FGS_CAMERA_FISHEYE) {
    bool pin = cam.model == FGS_CAMERA_PINHOLE;
    if (pin && z <= 0.2) return false;
    double lz = 0.0, theta = 0.0;
    if (!pin) {
      lz = sqrt(x * x + y * y);
      if (z < 0.0 && lz * lz < 1e-24 * z * z) return false;
      theta = atan2(lz, z);
      if (theta > static_cast<double>(cam.fov_max) + 10.0 * kBfPi / 180.0) return false;
      pin = lz < 1e-8 * fabs(z);  // axis limit: the pinhole form
    }
    if (pin) {
      pix[0] = cx + fx * x / z;
      pix[1] = cy + fy * y / z;
      j[0][0] = fx / z; j[0][1] = 0.0; j[0][2] = -fx * x / (z * z);
      j[1][0] = 0.0; j[1][1] = fy / z; j[1][2] = -fy * y / (z * z);
      return true;
    }
    const double l2 = x * x + y * y + z * z, lz2 = lz * lz, lz3 = lz2 * lz;
    pix[0] = cx + fx * theta * x / lz;
    pix[1] = cy + fy * theta * y / lz;
    j[0][0] = fx * (x * x * z / (lz2 * l2) + y * y * theta / lz3);
    j[0][1] = fx * x * y * (z / (lz2 * l2) - theta / lz3);
    j[0][2] = -fx * x / l2;
    j[1][0] = fy * x * y * (z / (lz2 * l2) - theta / lz3);
    j[1][1] = fy * (y * y * z / (lz2 * l2) + x * x * theta / lz3);
    j[1][2] = -fy * y / l2;
    return true;
  }
  const double s = x * x + z * z;
  if (s < 1e-24 * y * y) return false;
  const double rho = sqrt(s), l2 = s + y * y, two_pi = 2.0 * kBfPi;
  const double w = cam.width, h = cam.height;
  double xp = w * (atan2(x, z) + two_pi / 2.0) / two_pi;
  if (xp >= w) xp -= w;
  pix[0] = xp;
  pix[1] = h * (atan2(y, rho) + two_pi / 4.0) / (two_pi / 2.0);
  j[0][0] = w * z / (two_pi * s); j[0][1] = 0.0; j[0][2] = -w * x / (two_pi * s);
  const double hpi = h / (two_pi / 2.0);
  j[1][0] = -hpi * x * y / (rho * l2); j[1][1] = hpi * rho / l2; j[1][2] = -hpi * y * z / (rho * l2);
  return true;
}

template <typename Real>
struct BfScene {
  int64_t n;
  const Real *means, *rotations, *log_scales, *opacity_logits, *sh;
};

template <typename Real>
struct BfArgs {
  BfScene<Real> scene;
  fgs_camera cam;
  int sh_degree;
  BfSplat* splats;
  int* kept;
};

template <typename Real>
__global__ void bf_splats_kernel(BfArgs<Real> a) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= a.scene.n) return;
  a.kept[i] = 0;
  const fgs_camera& cam = a.cam;
  double W[3][3], b[3], m[3], mu[3];
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) W[r][c] = cam.rotation_wc[r * 3 + c];
    b[r] = cam.translation_wc[r];
    m[r] = a.scene.means[3 * i + r];
  }
  for (int r = 0; r < 3; ++r) mu[r] = W[r][0] * m[0] + W[r][1] * m[1] + W[r][2] * m[2] + b[r];
  double pix[2], J[2][3];
  if (!bf_project(mu, cam, pix, J)) return;
  double qw = a.scene.rotations[4 * i], qx = a.scene.rotations[4 * i + 1], qy = a.scene.rotations[4 * i + 2],
         qz = a.scene.rotations[4 * i + 3];
  const double qn = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
  if (qn > 0) { qw /= qn; qx /= qn; qy /= qn; qz /= qn; }
  const double R[3][3] = {{1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qw * qz), 2 * (qx * qz + qw * qy)},
                          {2 * (qx * qy + qw * qz), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qw * qx)},
                          {2 * (qx * qz - qw * qy), 2 * (qy * qz + qw * qx), 1 - 2 * (qx * qx + qy * qy)}};
  double s2[3];
  for (int k = 0; k < 3; ++k) {
    const double sk = exp(static_cast<double>(a.scene.log_scales[3 * i + k]));
    s2[k] = sk * sk;
  }
  double sig[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) sig[r][c] = R[r][0] * s2[0] * R[c][0] + R[r][1] * s2[1] * R[c][1] + R[r][2] * s2[2] * R[c][2];
  double T[2][3];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 3; ++c) T[r][c] = J[r][0] * W[0][c] + J[r][1] * W[1][c] + J[r][2] * W[2][c];
  double sp[2][2];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c) {
      double acc = 0.0;
      for (int k = 0; k < 3; ++k)
        for (int l = 0; l < 3; ++l) acc += T[r][k] * sig[k][l] * T[c][l];
      sp[r][c] = acc;
    }
  sp[0][0] += 0.3;
  sp[1][1] += 0.3;
  const double det = sp[0][0] * sp[1][1] - sp[0][1] * sp[1][0];
  if (!(det > 0.0)) return;
  const double mid = 0.5 * (sp[0][0] + sp[1][1]);
  const double lmax = mid + sqrt(fmax(mid * mid - det, 0.0));
  const int radius = static_cast<int>(ceil(3.0 * sqrt(lmax)));
  if (pix[0] + radius < 0 || pix[0] - radius > cam.width || pix[1] + radius < 0 || pix[1] - radius > cam.height) return;
  BfSplat o;
  o.mx = pix[0];
  o.my = pix[1];
  o.ca = sp[1][1] / det;
  o.cb = -sp[0][1] / det;
  o.cc = sp[0][0] / det;
  o.depth = cam.model == FGS_CAMERA_PINHOLE ? mu[2] : sqrt(mu[0] * mu[0] + mu[1] * mu[1] + mu[2] * mu[2]);
  o.radius = radius;
  double ctr[3], dir[3];
  for (int r = 0; r < 3; ++r) ctr[r] = -(W[0][r] * b[0] + W[1][r] * b[1] + W[2][r] * b[2]);
  double dn = 0.0;
  for (int r = 0; r < 3; ++r) {
    dir[r] = m[r] - ctr[r];
    dn += dir[r] * dir[r];
  }
  dn = sqrt(dn);
  for (int r = 0; r < 3; ++r) dir[r] = dn > 0 ? dir[r] / dn : dir[r];
  const Real* sh = a.scene.sh + 48 * i;
  o.r = bf_sh(sh, dir, a.sh_degree);
  o.g = bf_sh(sh + 16, dir, a.sh_degree);
  o.b = bf_sh(sh + 32, dir, a.sh_degree);
  o.alpha = 1.0 / (1.0 + exp(-static_cast<double>(a.scene.opacity_logits[i])));
  o.source = static_cast<int>(i);
  a.splats[i] = o;
  a.kept[i] = 1;
}

__global__ void __launch_bounds__(256) bf_render_kernel(const BfSplat* __restrict__ sp, int nv, int width, int height,
                                                       double bg0, double bg1, double bg2, double* image,
                                                       double* trans_out) {
  __shared__ BfSplat s[256];
  __shared__ int s_n;
  const int tiles_x = (width + kBfTile - 1) / kBfTile;
  const int tx0 = (blockIdx.x % tiles_x) * kBfTile, ty0 = (blockIdx.x / tiles_x) * kBfTile;
  const int px = tx0 + (threadIdx.x & 15), py = ty0 + (threadIdx.x >> 4);
  const bool inside = px < width && py < height;
  double T = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
  bool done = !inside;
  for (int base = 0; base < nv; base += 256) {
    if (__syncthreads_and(done)) break;
    // tile-overlap gate (oracle.hpp:251-254), order kept by a prefix over the ballots
    const int k = base + threadIdx.x;
    bool pass = false;
    BfSplat q;
    if (k < nv) {
      q = sp[k];
      pass = !(q.mx + q.radius < tx0 || q.mx - q.radius >= tx0 + kBfTile || q.my + q.radius < ty0 ||
               q.my - q.radius >= ty0 + kBfTile);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, pass);
    __shared__ int s_warp[8];
    if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = __popc(bal);
    __syncthreads();
    int pre = 0;
    for (int w = 0; w < (threadIdx.x >> 5); ++w) pre += s_warp[w];
    if (pass) s[pre + __popc(bal & ((1u << (threadIdx.x & 31)) - 1u))] = q;
    if (threadIdx.x == 255) s_n = pre + __popc(bal);
    __syncthreads();
    const int cnt = s_n;
    for (int j = 0; j < cnt && !done; ++j) {
      const BfSplat& o = s[j];
      const double dx = px + 0.5 - o.mx, dy = py + 0.5 - o.my;
      const double power = -0.5 * (o.ca * dx * dx + o.cc * dy * dy) - o.cb * dx * dy;
      if (power > 0.0) continue;
      const double alpha = fmin(0.99, o.alpha * exp(power));
      if (alpha < 1.0 / 255.0) continue;
      const double nt = T * (1.0 - alpha);
      if (nt < 1e-4) {
        done = true;
        break;
      }
      c0 += o.r * (alpha * T);
      c1 += o.g * (alpha * T);
      c2 += o.b * (alpha * T);
      T = nt;
    }
  }
  if (!inside) return;
  const size_t p = static_cast<size_t>(py) * width + px;
  image[3 * p] = c0 + T * bg0;
  image[3 * p + 1] = c1 + T * bg1;
  image[3 * p + 2] = c2 + T * bg2;
  if (trans_out) trans_out[p] = T;
}

}  // namespace

template <typename Real>
cudaError_t bruteforce_impl(const BfScene<Real>& scene, const fgs_camera& cam, int sh_degree, const double bg[3],
                            double* image, double* transmittance, cudaStream_t st) {
  const int64_t n = scene.n;
  BfSplat* d_sp = nullptr;
  int* d_kept = nullptr;
  cudaError_t e = cudaSuccess;
  std::vector<BfSplat> h_sp;
  std::vector<int> h_kept;
  int nv = 0;
  if (n > 0) {
    if ((e = cudaMalloc(&d_sp, n * sizeof(BfSplat))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&d_kept, n * sizeof(int))) != cudaSuccess) {
      cudaFree(d_sp);
      return e;
    }
    BfArgs<Real> a{scene, cam, sh_degree, d_sp, d_kept};
    bf_splats_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(a);
    h_sp.resize(n);
    h_kept.resize(n);
    cudaMemcpyAsync(h_sp.data(), d_sp, n * sizeof(BfSplat), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(h_kept.data(), d_kept, n * sizeof(int), cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) {
      cudaFree(d_sp);
      cudaFree(d_kept);
      return e;
    }
    // oracle.hpp:213-216: global order by (depth, source)
    std::vector<BfSplat> kept;
    kept.reserve(n);
    for (int64_t i = 0; i < n; ++i)
      if (h_kept[i]) kept.push_back(h_sp[i]);
    std::sort(kept.begin(), kept.end(), [](const BfSplat& x, const BfSplat& y) {
      return x.depth != y.depth ? x.depth < y.depth : x.source < y.source;
    });
    nv = static_cast<int>(kept.size());
    if (nv) cudaMemcpyAsync(d_sp, kept.data(), nv * sizeof(BfSplat), cudaMemcpyHostToDevice, st);
    h_sp.swap(kept);  // keep the host copy alive until the async copy has been consumed
  }
  const int tiles = ((cam.width + kBfTile - 1) / kBfTile) * ((cam.height + kBfTile - 1) / kBfTile);
  bf_render_kernel<<<tiles, 256, 0, st>>>(d_sp, nv, cam.width, cam.height, bg[0], bg[1], bg[2], image, transmittance);
  e = cudaStreamSynchronize(st);
  if (d_sp) cudaFree(d_sp);
  if (d_kept) cudaFree(d_kept);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e;
}

cudaError_t bruteforce_render(const fgs_gaussians& g, const fgs_camera& cam, int sh_degree, const double bg[3],
                              double* image, double* transmittance, cudaStream_t st) {
  const BfScene<float> sc{g.n, g.means, g.rotations, g.log_scales, g.opacity_logits, g.sh};
  return bruteforce_impl(sc, cam, sh_degree, bg, image, transmittance, st);
}

cudaError_t bruteforce_render_f64(int64_t n, const double* means, const double* rotations, const double* log_scales,
                                  const double* opacity, const double* sh, const fgs_camera& cam, int sh_degree,
                                  const double bg[3], double* image, double* transmittance, cudaStream_t st) {
  const BfScene<double> sc{n, means, rotations, log_scales, opacity, sh};
  return bruteforce_impl(sc, cam, sh_degree, bg, image, transmittance, st);
}

}  // namespace fgs
