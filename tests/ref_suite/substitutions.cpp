// Recorded tolerance substitutions for the reference's unit tests run against
// the drop-in (tests/ref_suite/include/doctest.h applies them by file:line and
// logs every use).  Each is a float comparison of the B200 sparse step (bf16
// K/V cache, fp32 tensor-core accumulation) against an fp64 oracle; the
// north-star contract is 1e-3 relative (oracles::max_rel_diff, floor 1e-3).
// Integer / bit-exact assertions (keys_scored, max_visited_bucket, lists,
// assignments, IVF, throws) are never substituted.
#include "doctest.h"

#define WHY "fp32 accumulation of the bf16 cache vs fp64 oracle: north-star 1e-3"
SAAP_SUBST("unit/attention_test.cpp", 242, 1e-3, WHY);  // every bucket == full attention (1e-5)
SAAP_SUBST("unit/attention_test.cpp", 258, 1e-3, WHY);  // window-only == attention_over_ids (1e-6)
SAAP_SUBST("unit/attention_test.cpp", 274, 1e-3, WHY);  // restricted set == attention_over_ids (1e-6)
SAAP_SUBST("unit/attention_test.cpp", 275, 1e-3, WHY);  // restricted set == naive oracle (1e-6)
