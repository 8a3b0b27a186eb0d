// Reference-side binding: a sketchtensor::ContractionEngine backed by the B200
// C-ABI (include/fcs_b200.h). This is the code a reference maintainer adds to
// proj/ to route SketchBackend::FCS to the GPU; it is
// compiled here against the reference's own headers (cpd.hpp:21-41) and
// tested against the reference FcsEngine by integration/test_drop_in.cpp.
#pragma once

#include <sketchtensor/cpd.hpp>

#include <cstddef>
#include <memory>
#include <vector>

#include "fcs_b200.h"

namespace sketchtensor_b200 {

class GpuFcsEngine final : public sketchtensor::ContractionEngine {
 public:
  // Engine ctor semantics of the chosen backend (cpd.cpp:36-197): sketch
  // backends build D = cfg.sketch_count sketches from families_for(t.shape(),
  // cfg) and drop the tensor; Plain keeps a device copy of it.
  GpuFcsEngine(const sketchtensor::DenseTensor& t, const sketchtensor::EstimatorConfig& cfg,
               sketchtensor::SketchBackend backend = sketchtensor::SketchBackend::FCS);
  ~GpuFcsEngine() override;
  GpuFcsEngine(const GpuFcsEngine&) = delete;
  GpuFcsEngine& operator=(const GpuFcsEngine&) = delete;

  double uvw(const Eigen::VectorXd& u, const Eigen::VectorXd& v,
             const Eigen::VectorXd& w) const override;
  Eigen::VectorXd iuv(const Eigen::VectorXd& a, const Eigen::VectorXd& b,
                      std::size_t free_mode) const override;
  void deflate(double weight, const Eigen::VectorXd& u, const Eigen::VectorXd& v,
               const Eigen::VectorXd& w) override;
  std::vector<std::size_t> shape() const override { return shape_; }

 private:
  st_engine* eng_ = nullptr;
  std::vector<std::size_t> shape_;
  double* dev_ = nullptr;  // device staging: 3 input vectors + 1 output
  std::size_t dev_len_ = 0;
};

// make_contraction_engine (cpd.cpp:220-232) with every backend on the GPU.
std::unique_ptr<sketchtensor::ContractionEngine> make_contraction_engine(
    const sketchtensor::DenseTensor& t, sketchtensor::SketchBackend backend,
    const sketchtensor::EstimatorConfig& cfg);

}  // namespace sketchtensor_b200
