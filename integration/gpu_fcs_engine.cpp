#include "gpu_fcs_engine.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <string>

namespace sketchtensor_b200 {

namespace {

// C-ABI status -> the reference's exception types.
void check(int rc) {
  if (rc == ST_OK) return;
  const std::string msg = st_last_error();
  if (rc == ST_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

GpuFcsEngine::GpuFcsEngine(const sketchtensor::DenseTensor& t,
                           const sketchtensor::EstimatorConfig& cfg,
                           sketchtensor::SketchBackend backend)
    : shape_(t.shape()) {
  if (t.order() != 3) throw std::invalid_argument("make_contraction_engine: order-3 tensor required");
  void* dt = nullptr;
  cuda_check(cudaMalloc(&dt, t.size() * sizeof(double)), "cudaMalloc");
  cuda_check(cudaMemcpy(dt, t.data().data(), t.size() * sizeof(double), cudaMemcpyHostToDevice),
             "cudaMemcpy");
  const int rc = st_engine_create_backend(&eng_, static_cast<int>(backend), ST_F64, dt,
                                          shape_.data(), cfg.hash_len, cfg.sketch_count, cfg.seed,
                                          nullptr);
  cudaFree(dt);
  check(rc);
  dev_len_ = *std::max_element(shape_.begin(), shape_.end());
  cuda_check(cudaMalloc(reinterpret_cast<void**>(&dev_), 4 * dev_len_ * sizeof(double)),
             "cudaMalloc");
}

GpuFcsEngine::~GpuFcsEngine() {
  st_engine_destroy(eng_);
  if (dev_) cudaFree(dev_);
}

double GpuFcsEngine::uvw(const Eigen::VectorXd& u, const Eigen::VectorXd& v,
                         const Eigen::VectorXd& w) const {
  const Eigen::VectorXd* in[3] = {&u, &v, &w};
  for (int n = 0; n < 3; ++n) {
    if (static_cast<std::size_t>(in[n]->size()) != shape_[n])
      throw std::invalid_argument("estimate_uvw: vector length mismatch");
    cuda_check(cudaMemcpy(dev_ + n * dev_len_, in[n]->data(), shape_[n] * sizeof(double),
                          cudaMemcpyHostToDevice), "cudaMemcpy");
  }
  check(st_engine_uvw(eng_, 1, dev_, dev_ + dev_len_, dev_ + 2 * dev_len_, dev_ + 3 * dev_len_, 1,
                      nullptr));
  double out = 0.0;
  cuda_check(cudaMemcpy(&out, dev_ + 3 * dev_len_, sizeof(double), cudaMemcpyDeviceToHost),
             "cudaMemcpy");
  return out;
}

Eigen::VectorXd GpuFcsEngine::iuv(const Eigen::VectorXd& a, const Eigen::VectorXd& b,
                                  std::size_t free_mode) const {
  if (free_mode > 2) throw std::invalid_argument("estimate_iuv: mode out of range");
  const std::size_t c1 = free_mode == 0 ? 1 : 0, c2 = free_mode == 2 ? 1 : 2;
  if (static_cast<std::size_t>(a.size()) != shape_[c1] ||
      static_cast<std::size_t>(b.size()) != shape_[c2])
    throw std::invalid_argument("estimate_iuv: vector length mismatch");
  cuda_check(cudaMemcpy(dev_, a.data(), a.size() * sizeof(double), cudaMemcpyHostToDevice),
             "cudaMemcpy");
  cuda_check(cudaMemcpy(dev_ + dev_len_, b.data(), b.size() * sizeof(double),
                        cudaMemcpyHostToDevice), "cudaMemcpy");
  check(st_engine_iuv(eng_, 1, dev_, dev_ + dev_len_, free_mode, dev_ + 3 * dev_len_, 1, nullptr));
  Eigen::VectorXd out(static_cast<Eigen::Index>(shape_[free_mode]));
  cuda_check(cudaMemcpy(out.data(), dev_ + 3 * dev_len_, shape_[free_mode] * sizeof(double),
                        cudaMemcpyDeviceToHost), "cudaMemcpy");
  return out;
}

void GpuFcsEngine::deflate(double weight, const Eigen::VectorXd& u, const Eigen::VectorXd& v,
                           const Eigen::VectorXd& w) {
  const Eigen::VectorXd* in[3] = {&u, &v, &w};
  for (int n = 0; n < 3; ++n)
    cuda_check(cudaMemcpy(dev_ + n * dev_len_, in[n]->data(), shape_[n] * sizeof(double),
                          cudaMemcpyHostToDevice), "cudaMemcpy");
  check(st_engine_deflate(eng_, weight, dev_, dev_ + dev_len_, dev_ + 2 * dev_len_, nullptr));
}

std::unique_ptr<sketchtensor::ContractionEngine> make_contraction_engine(
    const sketchtensor::DenseTensor& t, sketchtensor::SketchBackend backend,
    const sketchtensor::EstimatorConfig& cfg) {
  return std::make_unique<GpuFcsEngine>(t, cfg, backend);  // every backend runs on the GPU
}

}  // namespace sketchtensor_b200
