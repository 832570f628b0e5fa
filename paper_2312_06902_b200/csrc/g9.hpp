// G9: the synthetic 1F1B workload generator of SURVEY.md §8(d).
//
// Header-only, standard library only, so that the product library (bench
// inputs), the oracle and the reference driver (oracle/ref_driver.cpp) all
// draw bit-identical instances from the same libstdc++ std::mt19937 /
// distribution implementations.
//
//   * tau = 1000 us, quantum 1 us, blocking power 75 W;
//   * 9 frequencies 1410 - 75 j MHz, j = 0..8;
//   * stage s forward base b_s = B + eps_s (tau units), eps_s drawn from
//     uniform_int_distribution<int>(-1, 1) of mt19937(seed), one draw per
//     stage in stage order; the last stage is then overridden to
//     lround(B * imbalance); an optional straggler stage gets
//     b <- lround(b * phi);
//   * forward point j: time (b + j) tau, energy llround((b tau / 1e4) *
//     (4000 + 20000 * 1.25^-j)); backward point j: time (2b + 2j) tau,
//     energy 2 x the forward energy.
//
// Every profiled time is a tau multiple, so the frontier walk reaches T_min
// exactly and takes 24 (N + M - 1) steps.
#pragma once

#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

namespace pb_g9 {

inline constexpr std::int64_t kTau = 1000;
inline constexpr int kPoints = 9;

struct Point {
  int freq_mhz;
  std::int64_t time;
  std::int64_t energy;
};

struct Params {
  int stages = 4;
  int microbatches = 8;
  int base = 10;           // B, in tau units
  double imbalance = 1.2;  // last stage base = lround(B * imbalance)
  std::uint32_t seed = 1234;
  int straggler_stage = -1;  // -1: none
  double phi = 1.0;          // straggler slowdown
};

inline std::vector<int> stage_bases(const Params& p) {
  std::mt19937 rng(p.seed);
  std::vector<int> b(p.stages);
  for (int s = 0; s < p.stages; ++s) {
    std::uniform_int_distribution<int> eps(-1, 1);
    b[s] = p.base + eps(rng);
  }
  b[p.stages - 1] = static_cast<int>(std::lround(p.base * p.imbalance));
  if (p.straggler_stage >= 0 && p.straggler_stage < p.stages)
    b[p.straggler_stage] = static_cast<int>(std::lround(b[p.straggler_stage] * p.phi));
  return b;
}

// Points in strictly decreasing frequency (the reference's profile order).
inline std::vector<Point> stage_profile(int b, bool backward, std::int64_t tau = kTau) {
  std::vector<Point> pts;
  for (int j = 0; j < kPoints; ++j) {
    const double scale = static_cast<double>(b) * static_cast<double>(tau) / 1e4;
    const std::int64_t e =
        static_cast<std::int64_t>(std::llround(scale * (4000.0 + 20000.0 * std::pow(1.25, -j))));
    Point pt;
    pt.freq_mhz = 1410 - 75 * j;
    pt.time = backward ? (2 * static_cast<std::int64_t>(b) + 2 * j) * tau
                       : (static_cast<std::int64_t>(b) + j) * tau;
    pt.energy = backward ? 2 * e : e;
    pts.push_back(pt);
  }
  return pts;
}

// Config 5: instance i of the heterogeneous batch, drawn in this order from
// mt19937(1000 + i): N, M, imbalance, phi, straggler stage, profile seed.
inline Params batch_instance(int i) {
  std::mt19937 r(1000u + static_cast<std::uint32_t>(i));
  static const double kPhi[] = {1.0, 1.05, 1.1, 1.2, 1.3, 1.5};
  Params p;
  p.stages = std::uniform_int_distribution<int>(4, 16)(r);
  p.microbatches = std::uniform_int_distribution<int>(8, 256)(r);
  p.imbalance = std::uniform_real_distribution<double>(1.0, 1.25)(r);
  p.phi = kPhi[std::uniform_int_distribution<int>(0, 5)(r)];
  p.straggler_stage = std::uniform_int_distribution<int>(0, p.stages - 1)(r);
  p.seed = static_cast<std::uint32_t>(r());
  p.base = 10;
  return p;
}

// Named configs 1-4 of BASELINE.json (seed 1234).
inline Params named_config(int k, double phi = 1.0) {
  Params p;
  p.seed = 1234;
  switch (k) {
    case 1: p.stages = 4; p.microbatches = 8; p.base = 10; p.imbalance = 1.2; break;
    case 2: p.stages = 8; p.microbatches = 32; p.base = 10; p.imbalance = 1.2; break;
    case 3: p.stages = 8; p.microbatches = 128; p.base = 33; p.imbalance = 1.03; break;
    case 4:
      p.stages = 16; p.microbatches = 128; p.base = 10; p.imbalance = 1.10;
      if (phi != 1.0) { p.straggler_stage = 8; p.phi = phi; }
      break;
    default: break;
  }
  return p;
}

}  // namespace pb_g9
