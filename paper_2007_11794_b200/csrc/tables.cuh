// Container-level operations on one stream's device tables, for callers that
// drive the IndexTable / RescoreCache directly (the reference's fine-grained
// API; its own tests use it):
//   k_table_encode -- IndexTable.encode (context_table.py:76-89): content
//                     dedup (digest + byte compare), new index = len + 1
//   k_cache_get    -- RescoreCache.get (cache.py:80-94): counts lookups /
//                     hits / misses, enabled=False counts every lookup a miss
//   k_cache_put    -- RescoreCache.put (cache.py:96-108): first value wins
// The decoder and rnnlm_prob never use these: they resolve whole levels in
// assign_range with the same keys, digests and slot layout, so entries made
// here are found there and vice versa.  One thread walks the batch in call
// order (the reference's order); these calls are not a throughput path.
#pragma once

__global__ void k_table_encode(DevStreams S, uint32_t s, uint32_t n, const float *__restrict__ h,
                               const uint32_t *__restrict__ hist, const int32_t *__restrict__ hlen,
                               uint32_t *__restrict__ idx_out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int H = S.H;
    const uint64_t cb = (uint64_t)s * S.ct_cap;
    const uint32_t cmask = S.ct_cap - 1;
    for (uint32_t i = 0; i < n; i++) {
        const float *hi = h + (size_t)i * H;
        uint32_t meta[OTF_META];
        for (int k = 0; k < OTF_META; k++) meta[k] = 0;
        const int L = hlen[i];
        meta[0] = (uint32_t)L;
        for (int j = 0; j < L; j++) meta[1 + j] = hist[(size_t)i * S.order + j];
        unsigned long long dg = 0ull;                       // same digest as the decode path
        for (int u = 0; u < H; u++) dg += otf_dig_h((uint32_t)u, hi[u]);
        for (int k = 0; k < OTF_META; k++) dg += dig_meta(k, meta[k]);
        const unsigned long long key = otf_hash64(dg) | 1ull;
        uint32_t slot = (uint32_t)(key >> 20) & cmask, found = OTF_UNSET, free_slot = OTF_UNSET;
        for (uint32_t probes = 0; probes <= S.ct_cap; probes++) {
            const unsigned long long k = S.ct_key[cb + slot];
            if (k == 0ull) { free_slot = slot; break; }
            if (k == key) {
                const uint32_t row = S.ct_row[cb + slot];
                bool eq = true;
                for (int u = 0; u < H && eq; u++)
                    eq = __float_as_uint(S.arena_h[(size_t)row * H + u]) == __float_as_uint(hi[u]);
                for (int k2 = 0; k2 < OTF_META && eq; k2++) eq = S.arena_meta[(size_t)row * OTF_META + k2] == meta[k2];
                if (eq) { found = S.ct_idx[cb + slot]; break; }
            }
            slot = (slot + 1) & cmask;
        }
        if (found != OTF_UNSET) { idx_out[i] = found; continue; }
        const uint32_t tlen = S.table_len[s];
        if (free_slot == OTF_UNSET || tlen + 1 > S.max_ctx) { atomicOr(S.err, OTF_E_TABLE_FULL); return; }
        const uint32_t row = atomicAdd(S.arena_used, 1u);
        if (row >= S.arena_rows) { atomicOr(S.err, OTF_E_ARENA_FULL); return; }
        for (int u = 0; u < H; u++) S.arena_h[(size_t)row * H + u] = hi[u];
        for (int k = 0; k < OTF_META; k++) S.arena_meta[(size_t)row * OTF_META + k] = meta[k];
        const uint32_t idx = tlen + 1;
        S.ct_key[cb + free_slot] = key;
        S.ct_idx[cb + free_slot] = idx;
        S.ct_row[cb + free_slot] = row;
        S.ctx_row[(uint64_t)s * (S.max_ctx + 1) + idx] = row;
        S.table_len[s] = idx;
        idx_out[i] = idx;
    }
}

__device__ __forceinline__ uint32_t kc_find(const DevStreams &S, uint32_t s, unsigned long long key, bool *empty) {
    const uint64_t kb = (uint64_t)s * S.kc_cap;
    const uint32_t mask = S.kc_cap - 1;
    uint32_t sl = (uint32_t)otf_hash64(key) & mask;
    for (uint32_t probes = 0; probes <= S.kc_cap; probes++) {
        const unsigned long long k = S.kc_key[kb + sl];
        if (k == key) { *empty = false; return sl; }
        if (k == 0ull) { *empty = true; return sl; }
        sl = (sl + 1) & mask;
    }
    *empty = false;
    return OTF_UNSET;
}

__global__ void k_cache_get(DevStreams S, uint32_t s, uint32_t n, const uint32_t *__restrict__ c,
                            const int32_t *__restrict__ w, uint8_t *found, double *p, uint32_t *cn) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const uint64_t kb = (uint64_t)s * S.kc_cap;
    unsigned long long hits = 0;
    for (uint32_t i = 0; i < n; i++) {
        found[i] = 0; p[i] = 0.0; cn[i] = OTF_UNSET;
        if (!S.enabled) continue;
        bool empty;
        const uint32_t sl = kc_find(S, s, ((((unsigned long long)c[i]) << 32) | (uint32_t)w[i]) + 1ull, &empty);
        if (sl == OTF_UNSET || empty || S.kc_cnext[kb + sl] == OTF_UNSET) continue;
        found[i] = 1; p[i] = S.kc_p[kb + sl]; cn[i] = S.kc_cnext[kb + sl];
        hits++;
    }
    unsigned long long *stt = S.stats + (size_t)s * 8;
    stt[0] += n; stt[1] += hits; stt[2] += n - hits; stt[7] += n;
}

__global__ void k_cache_put(DevStreams S, uint32_t s, uint32_t n, const uint32_t *__restrict__ c,
                            const int32_t *__restrict__ w, const double *__restrict__ p,
                            const uint32_t *__restrict__ cn) {
    if (threadIdx.x != 0 || blockIdx.x != 0 || !S.enabled) return;
    const uint64_t kb = (uint64_t)s * S.kc_cap;
    for (uint32_t i = 0; i < n; i++) {
        const unsigned long long key = ((((unsigned long long)c[i]) << 32) | (uint32_t)w[i]) + 1ull;
        bool empty;
        const uint32_t sl = kc_find(S, s, key, &empty);
        if (sl == OTF_UNSET) { atomicOr(S.err, OTF_E_CACHE_FULL); return; }
        if (!empty && S.kc_cnext[kb + sl] != OTF_UNSET) continue;       // key in the cache: put is a no-op
        S.kc_key[kb + sl] = key;
        S.kc_claim[kb + sl] = OTF_UNSET;
        S.kc_p[kb + sl] = p[i];
        S.kc_cnext[kb + sl] = cn[i];
        S.stats[(size_t)s * 8 + 6] += 1;                                // resident entries
    }
}
