// The reference's operator and trainer test cases (proj/tests/test_model.cpp,
// proj/tests/test_trainer.cpp) run through the B200 binding
// (integration/d2ft_b200_trainer.cpp over libd2ft_b200.so), next to the
// unmodified reference library they compare against.
//
// Adapted, not copied: the reference's configs (d = 8, d/H = 4, T = 4) are
// below what the sm_100a kernels tile (d a multiple of 128, d/H in {32, 64}),
// so every case runs at d = 128; the reference's exact comparisons against
// its own fp64 arithmetic become the north_star tolerances (fp16 operands,
// fp32 accumulation: loss 1e-3 relative, gradients / updates 1e-2 normwise);
// bitwise properties of the schedule semantics (untouched bytes, frozen
// bases, fractions, engaged gradients) stay bitwise.
#include <cmath>
#include <cstring>

#include "doctest.h"
#include "d2ft/baselines.hpp"
#include "d2ft/model.hpp"
#include "d2ft/rng.hpp"
#include "d2ft/trainer.hpp"
#include "d2ft_b200_trainer.hpp"

using namespace d2ft;

namespace {

// test_trainer.cpp:16-27 at the B200 tile sizes (dh = 64, ffn slice 128)
ModelConfig trainer_config() {
  ModelConfig cfg;
  cfg.num_blocks = 2;
  cfg.heads_per_block = 2;
  cfg.model_dim = 128;
  cfg.ffn_hidden = 256;
  cfg.seq_len = 16;
  cfg.num_classes = 4;
  cfg.seed = 17;
  return cfg;
}

SynthDatasetSpec trainer_dataset_spec(const ModelConfig& cfg, int samples) {  // test_trainer.cpp:29-38
  SynthDatasetSpec spec;
  spec.num_samples = samples;
  spec.num_classes = cfg.num_classes;
  spec.token_dim = cfg.model_dim;
  spec.seq_len = cfg.seq_len;
  spec.noise_level = 0.4;
  spec.seed = 23;
  return spec;
}

TrainConfig base_train_config() {  // test_trainer.cpp:40-51
  TrainConfig tc;
  tc.epochs = 3;
  tc.learning_rate = 0.05;
  tc.momentum = 0.9;
  tc.batch_size = 10;
  tc.micro_batch_size = 2;  // 5 micro-batches per batch
  tc.seed = 3;
  tc.budget.n_full = 3;
  tc.budget.n_fwd = 1;
  return tc;
}

std::vector<std::uint8_t> block_bytes(const SubnetModel& m) {  // test_trainer.cpp:256-265
  std::vector<std::uint8_t> bytes;
  for (int r = 0; r < m.scheduled_count(); ++r)
    visit_tensors(m.subnet(1 + r), [&](const char*, const Matrix& mat) {
      const auto* p = reinterpret_cast<const std::uint8_t*>(mat.data.data());
      bytes.insert(bytes.end(), p, p + mat.data.size() * sizeof(double));
    });
  return bytes;
}

// max |a - b| / max |b| over the tensors of two subnets (engaged on both sides)
double normwise(const Subnet& a, const Subnet& b) {
  std::vector<const Matrix*> ta, tb;
  visit_tensors(a, [&](const char*, const Matrix& m) { ta.push_back(&m); });
  visit_tensors(b, [&](const char*, const Matrix& m) { tb.push_back(&m); });
  double worst = 0.0;
  for (size_t t = 0; t < ta.size(); ++t) {
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < ta[t]->data.size(); ++i) {
      num = std::max(num, std::abs(ta[t]->data[i] - tb[t]->data[i]));
      den = std::max(den, std::abs(tb[t]->data[i]));
    }
    if (den > 0) worst = std::max(worst, num / den);
  }
  return worst;
}

Matrix random_input(const ModelConfig& cfg, std::uint64_t seed) {  // test_model.cpp:30-35
  auto rng = make_rng(seed, 77);
  Matrix x(cfg.seq_len, cfg.model_dim);
  for (double& v : x.data) v = gaussian(rng);
  return x;
}

std::vector<OperationKind> all_full_column(const SubnetModel& m) {
  return std::vector<OperationKind>(static_cast<std::size_t>(m.scheduled_count()), OperationKind::Full);
}

}  // namespace

// ---------------------------------------------------------------- operator

TEST_CASE("device forward_backward matches the reference operator") {
  ModelConfig cfg = trainer_config();
  SubnetModel model(cfg);
  b200::DeviceModel dev(model, 4);
  auto rng = make_rng(41, 0);
  std::vector<Matrix> inputs;
  std::vector<int> labels;
  for (int i = 0; i < 3; ++i) {
    Matrix x(cfg.seq_len, cfg.model_dim);
    for (double& v : x.data) v = gaussian(rng);
    inputs.push_back(std::move(x));
    labels.push_back(i % cfg.num_classes);
  }
  for (auto col : {all_full_column(model),
                   std::vector<OperationKind>{OperationKind::Full, OperationKind::ForwardOnly,
                                              OperationKind::Shortcut, OperationKind::Full}}) {
    auto ref = model.forward_backward(inputs, labels, col);
    auto got = dev.forward_backward(inputs, labels, col);
    CHECK(std::abs(got.loss - ref.loss) <= 1e-3 * std::abs(ref.loss));
    REQUIRE(got.grads.size() == ref.grads.size());
    for (size_t si = 0; si < ref.grads.size(); ++si) {
      CHECK(got.grads[si].has_value() == ref.grads[si].has_value());
      if (ref.grads[si] && got.grads[si]) CHECK(normwise(*got.grads[si], *ref.grads[si]) <= 1e-2);
    }
  }
}

TEST_CASE("operation semantics inside the model loop") {  // test_model.cpp:326-369
  ModelConfig cfg = trainer_config();
  SubnetModel model(cfg);
  b200::DeviceModel dev(model, 2);
  Matrix input = random_input(cfg, 15);
  std::vector<Matrix> inputs = {input};
  std::vector<int> labels = {2};

  SUBCASE("gradients exist exactly for full-operation subnets") {
    auto col = all_full_column(model);
    col[0] = OperationKind::ForwardOnly;
    col[2] = OperationKind::Shortcut;
    auto fb = dev.forward_backward(inputs, labels, col);
    CHECK(fb.grads.front().has_value());  // embed always full
    CHECK(fb.grads.back().has_value());   // head always full
    CHECK(!fb.grads[1].has_value());      // p_o: no gradients
    CHECK(fb.grads[2].has_value());
    CHECK(!fb.grads[3].has_value());      // p_s
    CHECK(fb.grads[4].has_value());
  }

  SUBCASE("forward-only keeps the loss identical to full") {
    auto fb_full = dev.forward_backward(inputs, labels, all_full_column(model));
    auto col = all_full_column(model);
    col[1] = OperationKind::ForwardOnly;
    auto fb_mixed = dev.forward_backward(inputs, labels, col);
    CHECK(fb_full.loss == fb_mixed.loss);  // bitwise: identical activations
  }

  SUBCASE("all-shortcut blocks reduce to the embed-to-head path") {
    std::vector<OperationKind> col(static_cast<std::size_t>(model.scheduled_count()), OperationKind::Shortcut);
    auto fb = dev.forward_backward(inputs, labels, col);
    Matrix embed_out = model.subnet_forward(0, input, OperationKind::Full).y;
    Matrix logits = model.subnet_forward(model.subnet_count() - 1, embed_out, OperationKind::Full).y;
    double expected = cross_entropy(logits, labels[0], nullptr);
    CHECK(std::abs(fb.loss - expected) <= 1e-3 * std::abs(expected));
    for (int r = 0; r < model.scheduled_count(); ++r) CHECK(!fb.grads[1 + r].has_value());
  }

  SUBCASE("schedule column must cover every scheduled subnet") {
    std::vector<OperationKind> col(2, OperationKind::Full);
    CHECK_THROWS_AS(dev.forward_backward(inputs, labels, col), Error);
  }

  SUBCASE("logits match the reference inference path") {
    Matrix ref = model.logits(input);
    Matrix got = dev.logits(input);
    double den = 0.0, num = 0.0;
    for (int c = 0; c < cfg.num_classes; ++c) {
      den = std::max(den, std::abs(ref(0, c)));
      num = std::max(num, std::abs(got(0, c) - ref(0, c)));
    }
    CHECK(num <= 1e-2 * den);
  }
}

TEST_CASE("lora adapters on the device") {  // test_model.cpp:371-454
  ModelConfig cfg = trainer_config();

  SUBCASE("zero-initialized down matrices leave outputs bitwise unchanged") {
    SubnetModel base(cfg);
    SubnetModel with_lora(cfg);
    with_lora.attach_lora(2, 1.0);
    b200::DeviceModel db(base, 1), dl(with_lora, 1);
    Matrix x = random_input(cfg, 16);
    CHECK(db.logits(x).data == dl.logits(x).data);
  }

  SUBCASE("under lora only adapter tensors receive gradients") {
    SubnetModel model(cfg);
    model.attach_lora(2, 0.5);
    for (int r = 0; r < model.scheduled_count(); ++r) {
      Subnet& s = model.subnet(1 + r);
      auto rng = make_rng(60 + static_cast<std::uint64_t>(r), 0);
      for (double& v : s.lora->down_q.data) v = 0.1 * gaussian(rng);
      for (double& v : s.lora->down_k.data) v = 0.1 * gaussian(rng);
      for (double& v : s.lora->down_v.data) v = 0.1 * gaussian(rng);
    }
    b200::DeviceModel dev(model, 1);
    Matrix input = random_input(cfg, 17);
    std::vector<Matrix> inputs = {input};
    std::vector<int> labels = {0};
    auto fb = dev.forward_backward(inputs, labels, all_full_column(model));
    auto ref = model.forward_backward(inputs, labels, all_full_column(model));
    const Subnet& g = *fb.grads[1];
    double base_sum = 0.0, adapter_sum = 0.0;
    visit_tensors(g, [&](const char* name, const Matrix& m) {
      double s = 0.0;
      for (double v : m.data) s += std::abs(v);
      if (std::strncmp(name, "lora.", 5) == 0) adapter_sum += s;
      else base_sum += s;
    });
    CHECK(base_sum == 0.0);
    CHECK(adapter_sum > 0.0);
    for (int r = 0; r < model.scheduled_count(); ++r) CHECK(normwise(*fb.grads[1 + r], *ref.grads[1 + r]) <= 1e-2);
  }
}

// ---------------------------------------------------------------- trainer

TEST_CASE("standard policy reproduces the reference trainer") {  // test_trainer.cpp:156-250
  ModelConfig cfg = trainer_config();
  Dataset ds = make_synthetic_dataset(trainer_dataset_spec(cfg, 40));
  TrainConfig tc = base_train_config();
  tc.policy.kind = PolicyKind::Standard;
  SubnetModel ref_model(cfg), gpu_model(cfg);
  TrainHistory ref = train(ref_model, ds, tc);
  TrainHistory ours = b200::train(gpu_model, ds, tc);
  REQUIRE(ours.epochs.size() == ref.epochs.size());
  for (size_t e = 0; e < ref.epochs.size(); ++e) {
    if (std::abs(ours.epochs[e].loss - ref.epochs[e].loss) > 1e-3 * std::abs(ref.epochs[e].loss))
      std::printf("  epoch %zu: loss %.9g, reference %.9g\n", e, ours.epochs[e].loss, ref.epochs[e].loss);
    CHECK(std::abs(ours.epochs[e].loss - ref.epochs[e].loss) <= 1e-3 * std::abs(ref.epochs[e].loss));
    CHECK(ours.epochs[e].compute_fraction == 1.0);
    CHECK(ours.epochs[e].comm_fraction == 1.0);
  }
  for (int si = 0; si < cfg.num_blocks * cfg.heads_per_block + 2; ++si)
    CHECK(normwise(gpu_model.subnet(si), ref_model.subnet(si)) <= 1e-3);  // updated weights, fp32 path
}

TEST_CASE("d2ft policy: device schedule, pre-pass and step against the reference trainer") {
  ModelConfig cfg = trainer_config();
  Dataset ds = make_synthetic_dataset(trainer_dataset_spec(cfg, 40));
  TrainConfig tc = base_train_config();
  tc.policy.kind = PolicyKind::D2FT;
  tc.epochs = 2;
  SubnetModel ref_model(cfg), gpu_model(cfg);
  TrainHistory ref = train(ref_model, ds, tc);
  TrainHistory ours = b200::train(gpu_model, ds, tc);
  REQUIRE(ours.epochs.size() == ref.epochs.size());
  for (size_t e = 0; e < ref.epochs.size(); ++e) {
    // the budget fixes the realised fractions whatever the scores pick
    CHECK(ours.epochs[e].compute_fraction == ref.epochs[e].compute_fraction);
    CHECK(ours.epochs[e].comm_fraction == ref.epochs[e].comm_fraction);
    CHECK(std::isfinite(ours.epochs[e].loss));
  }
}

TEST_CASE("update locality under restrictive schedules") {  // test_trainer.cpp:252-295
  ModelConfig cfg = trainer_config();
  Dataset ds = make_synthetic_dataset(trainer_dataset_spec(cfg, 40));

  SUBCASE("all-shortcut blocks never change") {
    SubnetModel model(cfg);
    auto before = block_bytes(model);
    auto embed_before = model.subnet(0).w_embed.data;
    TrainConfig tc = base_train_config();
    tc.policy.kind = PolicyKind::Random;
    tc.budget.n_full = 0;
    tc.budget.n_fwd = 0;
    TrainHistory h = b200::train(model, ds, tc);
    CHECK(block_bytes(model) == before);
    CHECK(model.subnet(0).w_embed.data != embed_before);  // embed always trains
    CHECK(h.epochs.back().compute_fraction == 0.0);
    CHECK(h.epochs.back().comm_fraction == 0.0);
  }

  SUBCASE("forward-only cells accumulate exactly zero updates") {
    SubnetModel model(cfg);
    auto before = block_bytes(model);
    TrainConfig tc = base_train_config();
    tc.policy.kind = PolicyKind::Random;
    tc.budget.n_full = 0;
    tc.budget.n_fwd = 2;
    TrainHistory h = b200::train(model, ds, tc);
    CHECK(block_bytes(model) == before);
    CHECK(h.epochs.back().compute_fraction == 0.16);
    CHECK(h.epochs.back().comm_fraction == 0.2);
  }
}

TEST_CASE("realized cost fractions equal the scheduled budget exactly") {  // test_trainer.cpp:297-310
  ModelConfig cfg = trainer_config();
  Dataset ds = make_synthetic_dataset(trainer_dataset_spec(cfg, 40));
  SubnetModel model(cfg);
  TrainConfig tc = base_train_config();
  tc.policy.kind = PolicyKind::Random;
  tc.budget.n_full = 2;
  tc.budget.n_fwd = 1;
  TrainHistory h = b200::train(model, ds, tc);
  for (const EpochRecord& r : h.epochs) {
    CHECK(r.compute_fraction == 0.48);
    CHECK(r.comm_fraction == 0.5);
  }
}

TEST_CASE("evaluate") {  // test_trainer.cpp:312-339
  ModelConfig cfg = trainer_config();
  Dataset ds = make_synthetic_dataset(trainer_dataset_spec(cfg, 80));
  SubnetModel model(cfg);
  b200::DeviceModel dev(model, 16);
  const double got = b200::evaluate(dev, ds);
  const double ref = evaluate(model, ds);
  // argmax of fp16-operand logits may flip a near tie: at most 2 of 80
  CHECK(std::abs(got - ref) <= 2.0 / 80.0 + 1e-12);
  CHECK(b200::evaluate(dev, ds) == got);  // deterministic
}

TEST_CASE("policies run end to end and schedules stay feasible") {  // test_trainer.cpp:341-359
  ModelConfig cfg = trainer_config();
  Dataset ds = make_synthetic_dataset(trainer_dataset_spec(cfg, 40));
  for (PolicyKind kind : {PolicyKind::D2FT, PolicyKind::Random, PolicyKind::DPruningM, PolicyKind::DPruningMG,
                          PolicyKind::Scaler}) {
    SubnetModel model(cfg);
    TrainConfig tc = base_train_config();
    tc.policy.kind = kind;
    tc.policy.scaler = ScalerConfig::max();
    tc.epochs = 2;
    TrainHistory h = b200::train(model, ds, tc);
    CHECK(h.epochs.size() == 2);
    for (const EpochRecord& r : h.epochs) {
      CHECK(std::isfinite(r.loss));
      CHECK(r.compute_fraction <= 1.0);
    }
  }
}

TEST_CASE("training under a d2ft schedule reduces the loss") {  // test_trainer.cpp:361-370
  ModelConfig cfg = trainer_config();
  Dataset ds = make_synthetic_dataset(trainer_dataset_spec(cfg, 40));
  SubnetModel model(cfg);
  TrainConfig tc = base_train_config();
  tc.policy.kind = PolicyKind::D2FT;
  tc.epochs = 6;
  TrainHistory h = b200::train(model, ds, tc);
  CHECK(h.epochs.back().loss < h.epochs.front().loss);
}

TEST_CASE("lora training freezes every base parameter bit") {  // test_trainer.cpp:372-387
  ModelConfig cfg = trainer_config();
  Dataset ds = make_synthetic_dataset(trainer_dataset_spec(cfg, 40));
  SubnetModel model(cfg);
  model.attach_lora(2, 1.0);
  auto base_before = model.parameter_bytes(/*include_adapters=*/false);
  auto all_before = model.parameter_bytes(true);
  TrainConfig tc = base_train_config();
  tc.policy.kind = PolicyKind::D2FT;
  tc.cost_model = CostModel::lora_finetune();
  tc.epochs = 3;
  b200::train(model, ds, tc);
  CHECK(model.parameter_bytes(false) == base_before);
  CHECK(model.parameter_bytes(true) != all_before);  // the adapters moved
}

TEST_CASE("infeasible budgets fail before touching the model") {  // test_trainer.cpp:389-400
  ModelConfig cfg = trainer_config();
  Dataset ds = make_synthetic_dataset(trainer_dataset_spec(cfg, 40));
  SubnetModel model(cfg);
  auto before = model.parameter_bytes();
  TrainConfig tc = base_train_config();
  tc.budget.n_full = 5;
  tc.budget.n_fwd = 2;  // 7 > 5 micro-batches
  CHECK_THROWS_AS(b200::train(model, ds, tc), Error);
  CHECK(model.parameter_bytes() == before);
}

TEST_CASE("non-finite gradients are rejected") {  // test_trainer.cpp:150-153 (sgd_momentum_step)
  ModelConfig cfg = trainer_config();
  Dataset ds = make_synthetic_dataset(trainer_dataset_spec(cfg, 40));
  ds.samples[7](3, 5) = std::nan("");
  SubnetModel model(cfg);
  TrainConfig tc = base_train_config();
  tc.policy.kind = PolicyKind::Standard;
  CHECK_THROWS_AS(b200::train(model, ds, tc), Error);
}
