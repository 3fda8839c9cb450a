// temporary stubs (replaced by hlu.cu)
#include "hmatrix.h"
std::string stats_to_json(const std::map<std::string, double>& m);
std::string hmat_stats(const cbie_hmat* h);
extern "C" {
int cbie_hlu_factor(cbie_hmat*, double, cbie_hlu**) { return CBIE_ESTATE; }
void cbie_hlu_destroy(cbie_hlu*) {}
int cbie_hlu_solve(cbie_hlu*, const cbie_c128*, cbie_c128*, int) { return CBIE_ESTATE; }
int cbie_stats_json(const void* h, int which, char* buf, size_t cap) {
  if (!h || !buf || cap == 0) return CBIE_EINVALID;
  std::string s = which == 0 ? stats_to_json(((const cbie_ctx*)h)->stat)
                             : which == 1 ? hmat_stats((const cbie_hmat*)h) : "{}";
  if (s.size() + 1 > cap) return CBIE_EINVALID;
  memcpy(buf, s.c_str(), s.size() + 1);
  return CBIE_OK;
}
}
