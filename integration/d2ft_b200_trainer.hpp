// Reference-side binding of the operator and trainer API (core/include/d2ft/
// model.hpp, trainer.hpp) over the B200 engine C-ABI (include/d2ft_b200_engine.h).
//
// d2ft::b200::DeviceModel is SubnetModel's compute on one B200: the same
// forward_backward signature and result (model.hpp:206-211, 252-254; grads
// engaged exactly for embed, head and the Full block subnets) with the
// parameters resident on the device.  d2ft::b200::train is train()
// (trainer.hpp:94-99, trainer.cpp:158-305) with the batch body on the device:
// the fp64 Dataset samples are gathered H2D per batch, the D2FT policy's
// knapsack runs inside the step, every other policy's table goes through the
// explicit-codes step.  A maintainer calls these where trainer.cpp /
// scoring.cpp call SubnetModel::forward_backward and train.
#pragma once

#include <span>
#include <vector>

#include "d2ft/data.hpp"
#include "d2ft/model.hpp"
#include "d2ft/trainer.hpp"
#include "d2ft_b200.h"
#include "d2ft_b200_engine.h"

namespace d2ft::b200 {

class DeviceModel {
 public:
  /// Uploads `host`'s parameters (and LoRA adapters when attached); velocity 0.
  DeviceModel(const SubnetModel& host, int max_batch);
  ~DeviceModel();
  DeviceModel(const DeviceModel&) = delete;
  DeviceModel& operator=(const DeviceModel&) = delete;

  /// model.cpp:416-520 on the device: loss = mean CE over the micro-batch,
  /// grads[i] engaged for embed, head and Full block subnets (zero tensors
  /// of the embed/head in LoRA mode, adapter gradients only, as the reference).
  ForwardBackwardResult forward_backward(std::span<const Matrix> inputs, std::span<const int> labels,
                                         std::span<const OperationKind> schedule_column) const;
  /// SubnetModel::logits for one sample (every subnet active).
  Matrix logits(const Matrix& input) const;

  void upload(const SubnetModel& host);      // parameters (+ adapters); zeroes the velocity
  /// Device parameters -> host tensors (canonical order).  `touched` (one flag
  /// per subnet, may be null = all) limits the write to subnets the device
  /// updated, so untouched subnets keep their exact fp64 bytes (the device
  /// holds fp32 masters); in LoRA mode only adapter tensors are written.
  void download(SubnetModel& host, const std::vector<char>* touched = nullptr) const;
  d2ft_engine* engine() const { return eng_; }
  const ModelConfig& config() const { return shape_.config(); }
  int max_batch() const { return max_batch_; }

 private:
  SubnetModel shape_;  // zero-initialised copy of the host model's layout (grads_like)
  d2ft_engine* eng_ = nullptr;
  int max_batch_ = 0;
  bool lora_ = false;
};

/// train() (trainer.cpp:158-305) with the batch body on the B200: scoring
/// pre-pass on the device, per-batch schedule (the D2FT knapsack inside the
/// step; Standard / Random / Scaler / pruning tables through the
/// explicit-codes step), fp64 Dataset samples gathered per batch with the
/// next batch prefetched, SGD-momentum on the touched subnets.  `model`
/// receives the trained parameters at every epoch end; EpochRecord fields as
/// the reference (top1 = evaluate on the device).
TrainHistory train(SubnetModel& model, const Dataset& dataset, const TrainConfig& config);

/// evaluate() (trainer.cpp:307-319) through DeviceModel::logits.
double evaluate(const DeviceModel& model, const Dataset& dataset);

}  // namespace d2ft::b200
