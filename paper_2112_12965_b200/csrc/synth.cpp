// synth.cpp -- seeded synthetic inputs for the BASELINE configurations
// (host C++, std::mt19937_64 + <random> distributions, like the reference's
// tests/synth.hpp:19-45). Built as libtsd_synth.so; used by bench.py and the
// tests to generate inputs on the host so the GPU path and the CPU
// oracle/reference always consume the same arrays.
//
//  walk     cumulative sum of N(0,1) draws with one distribution object per
//           call (same draw discipline as the reference's synth::walk)
//  ecg      BASELINE C2/C3: beats of 5 Gaussian bumps (P,Q,R,S,T), per-bump
//           amplitude x U(0.9,1.1), period U{240..260}, + N(0,0.05); optional
//           anomalous beats with the R bump inverted and widened 2x
//  traffic  BASELINE C5: period-288 sinusoid + half-amplitude period-2016
//           sinusoid + N(0,0.2) + random level shifts
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <random>
#include <vector>

namespace {

using rng_t = std::mt19937_64;

void walk(rng_t& rng, size_t n, double* out) {
  std::normal_distribution<double> g(0.0, 1.0);
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) {
    s += g(rng);
    out[i] = s;
  }
}

void noise(rng_t& rng, size_t n, double* out) {
  std::normal_distribution<double> g(0.0, 1.0);
  for (size_t i = 0; i < n; ++i) out[i] = g(rng);
}

struct Bump {
  double c, w, a;
};
// P, Q, R, S, T wave template (centre, width as a fraction of the beat; amplitude)
const Bump kBeat[5] = {{0.20, 0.025, 0.25}, {0.45, 0.008, -0.35}, {0.50, 0.012, 1.60}, {0.55, 0.008, -0.30},
                       {0.75, 0.040, 0.45}};

}  // namespace

extern "C" {

void* tsd_rng_new(uint64_t seed) { return new rng_t(seed); }
void tsd_rng_free(void* h) { delete static_cast<rng_t*>(h); }
void tsd_rng_walk(void* h, size_t n, double* out) { walk(*static_cast<rng_t*>(h), n, out); }
void tsd_rng_noise(void* h, size_t n, double* out) { noise(*static_cast<rng_t*>(h), n, out); }

void tsd_synth_walk(uint64_t seed, size_t n, double* out) {
  rng_t rng(seed);
  walk(rng, n, out);
}

// `count` independent walks of `len` samples drawn back to back from one seed
void tsd_synth_walks(uint64_t seed, size_t count, size_t len, double* out) {
  rng_t rng(seed);
  for (size_t k = 0; k < count; ++k) walk(rng, len, out + k * len);
}

void tsd_synth_sine(size_t n, double period, double amp, double* out) {
  for (size_t i = 0; i < n; ++i) out[i] = amp * std::sin(2.0 * M_PI * static_cast<double>(i) / period);
}

// ECG-like pulse train of n samples. n_anom anomalous beats are placed at
// distinct random beats (not the first/last two); their start samples are
// written to anom_starts (sorted) when non-null. Returns the beat count.
size_t tsd_synth_ecg(uint64_t seed, size_t n, size_t n_anom, double* out, size_t* anom_starts) {
  rng_t rng(seed);
  std::uniform_int_distribution<int> period(240, 260);
  std::uniform_real_distribution<double> jit(0.9, 1.1);
  std::normal_distribution<double> g(0.0, 0.05);
  std::vector<size_t> starts, lens;
  for (size_t at = 0; at < n;) {
    const size_t p = static_cast<size_t>(period(rng));
    starts.push_back(at);
    lens.push_back(p);
    at += p;
  }
  const size_t nb = starts.size();
  std::vector<char> anom(nb, 0);
  if (n_anom > 0 && nb > 4) {
    std::vector<size_t> cand(nb - 4);
    std::iota(cand.begin(), cand.end(), size_t(2));
    std::shuffle(cand.begin(), cand.end(), rng);
    for (size_t k = 0; k < n_anom && k < cand.size(); ++k) anom[cand[k]] = 1;
  }
  size_t na = 0;
  for (size_t b = 0; b < nb; ++b) {
    double amp[5];
    for (int k = 0; k < 5; ++k) amp[k] = kBeat[k].a * jit(rng);
    double wr = kBeat[2].w;
    if (anom[b]) {
      amp[2] = -amp[2];
      wr *= 2.0;
      if (anom_starts) anom_starts[na] = starts[b];
      ++na;
    }
    const double P = static_cast<double>(lens[b]);
    for (size_t i = 0; i < lens[b] && starts[b] + i < n; ++i) {
      const double t = static_cast<double>(i) / P;
      double v = 0.0;
      for (int k = 0; k < 5; ++k) {
        const double w = k == 2 ? wr : kBeat[k].w;
        const double z = (t - kBeat[k].c) / w;
        v += amp[k] * std::exp(-0.5 * z * z);
      }
      out[starts[b] + i] = v;
    }
  }
  for (size_t i = 0; i < n; ++i) out[i] += g(rng);
  return nb;
}

// nseries transportation-like daily-periodic series of len samples each
void tsd_synth_traffic(uint64_t seed, size_t nseries, size_t len, double* out) {
  rng_t rng(seed);
  std::uniform_real_distribution<double> u01(0.0, 1.0);
  std::normal_distribution<double> g(0.0, 1.0);
  for (size_t s = 0; s < nseries; ++s) {
    const double A = 0.8 + 0.4 * u01(rng);
    const double ph = 288.0 * u01(rng), phw = 2016.0 * u01(rng);
    double level = g(rng);
    double* x = out + s * len;
    for (size_t t = 0; t < len; ++t) {
      if (u01(rng) < 1.0 / 1500.0) level += g(rng);  // random level shift
      const double tt = static_cast<double>(t);
      x[t] = A * std::sin(2.0 * M_PI * (tt + ph) / 288.0) + 0.5 * A * std::sin(2.0 * M_PI * (tt + phw) / 2016.0) +
             level + 0.2 * g(rng);
    }
  }
}

}  // extern "C"
