// geometry.cuh -- per-sample source geometry of the variable-size dataset
// (BASELINE configs[4], cfg5): sample id is H x W x 3 u8 HWC with
// H, W = 128 + bounded(385) drawn from SplitMix64(derive_seed(data_seed, id, 1))
// (oracle: lo_sample_hw).  In HBM each row is padded to a 4-byte pitch
// (var_pitch) and each sample to 16 bytes, so every row starts word aligned and
// a bilinear tap's byte phase is a per-column constant (augment.cu K7); every
// learner computes the same global prefix of padded sizes, so a sample's
// offset inside its owner's shard is prefix[s] - prefix[first(owner)].
#pragma once
#include <cstdint>

#include "locload_b200.h"
#include "locload_rng.cuh"

namespace ll {

constexpr uint32_t kVarMin = 128;
constexpr uint32_t kVarSpan = 385;  // H, W in [128, 512]

LL_HD void var_hw(uint64_t data_seed, uint64_t id, uint32_t* h, uint32_t* w) {
    SplitMix r(derive_seed(data_seed, id, 1));
    *h = kVarMin + static_cast<uint32_t>(r.bounded(kVarSpan));
    *w = kVarMin + static_cast<uint32_t>(r.bounded(kVarSpan));
}

LL_HD uint64_t pad16(uint64_t b) { return (b + 15) & ~15ull; }

// HBM row pitch of a W-pixel u8 RGB row, and the padded bytes of an H x W sample
LL_HD uint32_t var_pitch(uint32_t w) { return (3u * w + 3u) & ~3u; }
LL_HD uint64_t var_bytes(uint32_t h, uint32_t w) {
    return pad16(static_cast<uint64_t>(h) * var_pitch(w));
}

// Per-sample augment parameters (oracle lo_aug_params_for):
// stream SplitMix64(derive_seed(seed, epoch, id)); crop (ch, cw) = the output
// size (LL_AUG_CROP) or the largest square min(H, W) (LL_AUG_RESIZE);
// y0 = bounded(H - ch + 1), x0 = bounded(W - cw + 1), flip = next() >> 63.
struct Params {
    uint32_t y0, x0, ch, cw, flip;
};

LL_HD Params aug_params(uint64_t seed, uint64_t epoch, uint64_t id, uint32_t H, uint32_t W,
                        uint32_t out_h, uint32_t out_w, int mode) {
    Params q;
    if (mode == LL_AUG_CROP) {
        q.ch = out_h;
        q.cw = out_w;
    } else {
        q.ch = q.cw = H < W ? H : W;
    }
    SplitMix r(derive_seed(seed, epoch, id));
    q.y0 = static_cast<uint32_t>(r.bounded(static_cast<uint64_t>(H - q.ch) + 1));
    q.x0 = static_cast<uint32_t>(r.bounded(static_cast<uint64_t>(W - q.cw) + 1));
    q.flip = static_cast<uint32_t>(r.next() >> 63);
    return q;
}

} // namespace ll
