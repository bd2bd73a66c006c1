#include "plant.h"

#include <cmath>

namespace dd {

namespace {
uint64_t mix(uint64_t seed, uint64_t m) {
    uint64_t z = seed + m * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
uint64_t derive(uint64_t base, uint64_t index) {
    uint64_t z = base + (index + 1) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 30)) * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
}  // namespace

PlantTable make_plant_table(int vocab, int d, const dd_plant_desc* plant) {
    PlantTable t;
    t.emb_std = (plant && plant->emb_std > 0.0f) ? plant->emb_std : 0.02f;
    t.src.assign(vocab, -1);
    t.perm.resize(vocab);
    for (int i = 0; i < vocab; ++i) t.perm[i] = i;
    if (!plant || !(plant->alpha > 0.0)) return t;
    uint64_t counter = 0;
    for (int i = vocab - 1; i >= 1; --i) {
        const uint64_t j = mix(plant->plant_seed, ++counter) % static_cast<uint64_t>(i + 1);
        const int32_t tmp = t.perm[i];
        t.perm[i] = t.perm[j];
        t.perm[j] = tmp;
    }
    const uint64_t sel = derive(plant->plant_seed, 1);
    for (int tok = 0; tok < vocab; ++tok) {
        const double u =
            static_cast<double>(mix(sel, static_cast<uint64_t>(tok) + 1) >> 11) * 0x1.0p-53;
        if (u < plant->alpha) {
            t.src[t.perm[tok]] = tok;
            t.any = true;
        }
    }
    t.coef = static_cast<float>(static_cast<double>(plant->gain) /
                                (static_cast<double>(t.emb_std) * std::sqrt(static_cast<double>(d))));
    return t;
}

}  // namespace dd
