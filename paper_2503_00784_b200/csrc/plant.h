// Planted shared-bigram structure for synthetic random-init weights
// (SURVEY.md §7 hard part 1).  Target and draft are generated from different
// weight seeds but the same plant: for a fraction alpha of tokens t, the LM-head
// row of pi(t) gets coef * E[t] added, so both models put a large logit on
// pi(t) after seeing t.  alpha = 0 is pure random init.
#pragma once

#include <stdint.h>

#include <vector>

#include "../../include/duodec_b200.h"

namespace dd {

struct PlantTable {
    bool any = false;
    float emb_std = 0.02f;
    float coef = 0.0f;          // gain / (emb_std * sqrt(d))
    std::vector<int32_t> src;   // src[v] = t with pi(t) = v and t planted, else -1
    std::vector<int32_t> perm;  // pi
};

// pi: Fisher-Yates driven by RandomStream(plant_seed) draws; planted(t):
// uniform(derive_seed(plant_seed, 1), draw t+1) < alpha.  Same recipe in
// oracle/llama_ref.c.
PlantTable make_plant_table(int vocab, int d, const dd_plant_desc* plant);

}  // namespace dd
