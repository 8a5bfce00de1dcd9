// Persistent whole-iteration engine (placeholder plan; see solver.cu).
#pragma once
namespace scfr {
struct PersistentPlan {
    int ctas = 0;
};
}  // namespace scfr
