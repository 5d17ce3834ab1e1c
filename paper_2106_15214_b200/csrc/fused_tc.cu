// Fused single-read fp32 pass (tcgen05 / TMEM / TMA) -- see DESIGN.md.
// Placeholder until the tensor-core kernel lands: reports "unsupported" so
// the engine uses the reference-order schedule.
#include "engine.h"

namespace bnmf {

struct FusedState { int dummy; };

bool fused_supported(int, int, int, int, int, int, int, double) { return false; }
int fused_create(FusedState** out, const FusedIO&, std::string& err) {
  *out = nullptr; err = "fused pass not built"; return -1;
}
int fused_begin(FusedState*, const FusedIO&, std::string& err) { err = "fused pass not built"; return -1; }
int fused_enqueue_iteration(FusedState*, const FusedIO&, int, std::string& err) {
  err = "fused pass not built"; return -1;
}
int fused_export(FusedState*, const FusedIO&, std::string&) { return 0; }
void fused_destroy(FusedState* fs) { delete fs; }

}  // namespace bnmf
