// Reference output formats (driver.cpp:131-215): the solver log rows and the
// energy-reduction table, so a GPU run writes the same artifacts as the CLI.
#include <cstdio>

#include "../../include/parorb_gpu.h"

extern "C" {

int po_format_log_row(const po_record* r, char* buf, int len) {  // driver.cpp:136-142
  if (!r || !buf || len <= 0) return -1;
  const int n = std::snprintf(buf, (size_t)len, "%d,%d,%.17g,%.17g,%.17g,%d,%d,%d,%.17g,%.3f",
                              r->level, r->iter, r->energy, r->grad_norm, r->tau, r->backtracks,
                              r->did_orth ? 1 : 0, r->did_diag ? 1 : 0, r->offdiag_max,
                              r->wall_ms);
  return n < len ? n : -1;
}

int po_write_log(const char* path, const po_record* recs, int n, int log_every) {
  if (!path || (n > 0 && !recs) || log_every < 1) return PO_EINVAL;
  FILE* f = std::fopen(path, "w");
  if (!f) return PO_EINVAL;
  std::fprintf(f, "level,iter,energy,grad_norm,tau,backtracks,did_orth,did_diag,offdiag_max,wall_ms\n");
  char buf[320];
  for (int i = 0; i < n; ++i) {
    const bool last_of_level = i + 1 == n || recs[i + 1].level != recs[i].level;
    if (recs[i].iter % log_every == 0 || last_of_level) {
      po_format_log_row(&recs[i], buf, sizeof buf);
      std::fprintf(f, "%s\n", buf);
    }
  }
  const bool ok = std::ferror(f) == 0;
  return std::fclose(f) == 0 && ok ? PO_OK : PO_EINVAL;
}

int po_write_reduction(const char* path, const po_record* recs, int n, double e_min) {
  if (!path || (n > 0 && !recs)) return PO_EINVAL;
  FILE* f = std::fopen(path, "w");
  if (!f) return PO_EINVAL;
  std::fprintf(f, "iter,energy_minus_emin\n");
  int final_level = 0;
  for (int i = 0; i < n; ++i) final_level = recs[i].level > final_level ? recs[i].level : final_level;
  for (int i = 0; i < n; ++i)
    if (recs[i].level == final_level && recs[i].did_orth)
      std::fprintf(f, "%d,%.17g\n", recs[i].iter, recs[i].energy - e_min);
  const bool ok = std::ferror(f) == 0;
  return std::fclose(f) == 0 && ok ? PO_OK : PO_EINVAL;
}

}  // extern "C"
