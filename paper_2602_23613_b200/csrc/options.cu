// Per-handle options and allocation pool (see Options in common.cuh).
#include <cstring>
#include <string>

#include "common.cuh"

namespace hcamg {

namespace {
thread_local const Options* t_opts = nullptr;
thread_local cudaMemPool_t t_pool = nullptr;

int64_t env_i(const char* k, int64_t d) {
  const char* v = getenv(k);
  return v && *v ? atoll(v) : d;
}
}  // namespace

// Round 1 selected these paths with process-wide environment variables; they
// still seed a new handle's defaults so existing scripts keep working.
Options options_from_env() {
  Options o;
  if (const char* e = getenv("HCAMG_SWEEP")) {
    const std::string m(e);
    o.sweep = m == "leg" || m == "cluster" ? SWEEP_LEG : m == "grid" ? SWEEP_GRID : m == "wave" ? SWEEP_WAVE
              : m == "flow" ? SWEEP_FLOW : m == "fwave" ? SWEEP_FWAVE : SWEEP_AUTO;
  }
  o.giant_min = env_i("HCAMG_GIANT_MIN", o.giant_min);
  o.coarse_gemv_min = env_i("HCAMG_COARSE_GEMV_MIN", o.coarse_gemv_min);
  o.coarse_symv = (int)env_i("HCAMG_COARSE_SYMV", o.coarse_symv);
  if (const char* e = getenv("HCAMG_PAPPLY")) o.factor_apply = std::string(e) != "z";
  o.form_z = (int)env_i("HCAMG_FORM_Z", o.form_z);
  o.tri_calib = (int)env_i("HCAMG_TRI_CALIB", o.tri_calib);
  return o;
}

const Options& opts() {
  static const Options defaults = options_from_env();
  return t_opts ? *t_opts : defaults;
}

OptionsScope::OptionsScope(const Options* o) : prev(t_opts) { t_opts = o; }
OptionsScope::~OptionsScope() { t_opts = prev; }

namespace {
thread_local double t_flops = 0.0;
}
void count_flops(double f) { t_flops += f; }
double StageTimer::peek_flops() { return t_flops; }
double take_flops() {
  const double f = t_flops;
  t_flops = 0.0;
  return f;
}

PoolScope::PoolScope(cudaMemPool_t p) : prev(t_pool) { t_pool = p; }
PoolScope::~PoolScope() { t_pool = prev; }
cudaMemPool_t current_pool() { return t_pool; }

}  // namespace hcamg
