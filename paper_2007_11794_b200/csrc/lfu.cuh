// lfu.cuh -- capacity-bounded RescoreCache (cache.py:61-134), included by
// capi.cu after struct OtflmStreams.
//
// The reference's bounded cache evicts the entry with the smallest
// (use count, last use) -- LFU with LRU tie-break, a lazy heap in
// cache.py:98-128.  Whether a lookup hits depends only on the sequence of
// keys, never on the values (p and c' are pure functions of (c, w); a
// recomputed entry deduplicates to the same context index), so the device
// decodes exactly as in unbounded mode and assign_range logs every stream's
// lookups in reference order (kc slot + whether the device computed it).
// k_lfu_replay then runs the policy over the log with the O(1) LFU structure
// (a list of frequency nodes in ascending order, each holding its entries in
// last-use order: evicting the head of the first node = argmin (freq, last
// use)), one thread per stream, and rewrites the window's hit / miss
// counters, the resident entry count and the eviction counters.
//
// The cache VALUES of evicted keys stay memoised in the device table (the
// policy models the reference's host-memory bound; HBM holds the memo), so a
// policy miss on an evicted key costs no recomputation here.

#define LFU_NIL 0xFFFFFFFFu

struct DevLfu {
    int S;
    uint32_t E;                      // allocated entries per stream (pitch)
    uint32_t cap;                    // allowed resident entries (<= E)
    uint32_t kc_cap;
    uint32_t *kc_lfu;                // [S][kc_cap] entry of a resident key
    uint32_t *en_slot, *en_prev, *en_next, *en_f;           // [S][E]
    uint32_t *fn_freq, *fn_prev, *fn_next, *fn_head, *fn_tail;   // [S][E + 1]
    uint32_t *sc;                    // [S][8] first fnode, n_res, en_bump, en_free, fn_bump, fn_free
    unsigned long long *ev;          // [S][2] evictions: window, rolled
};

struct LfuHost {
    DevLfu d{};
    Allocs mem;
};

namespace lfu {
struct View {
    uint32_t *kc_lfu, *en_slot, *en_prev, *en_next, *en_f, *fn_freq, *fn_prev, *fn_next, *fn_head, *fn_tail, *sc;
    __device__ View(const DevLfu &L, int s) {
        const size_t e = (size_t)s * L.E, f = (size_t)s * (L.E + 1);
        kc_lfu = L.kc_lfu + (size_t)s * L.kc_cap;
        en_slot = L.en_slot + e; en_prev = L.en_prev + e; en_next = L.en_next + e; en_f = L.en_f + e;
        fn_freq = L.fn_freq + f; fn_prev = L.fn_prev + f; fn_next = L.fn_next + f;
        fn_head = L.fn_head + f; fn_tail = L.fn_tail + f;
        sc = L.sc + (size_t)s * 8;
    }
    // scalars: sc[0] first fnode, sc[1] resident, sc[2] entry bump, sc[3] entry free list,
    //          sc[4] fnode bump, sc[5] fnode free list
    __device__ uint32_t alloc_en() {
        uint32_t e = sc[3];
        if (e != LFU_NIL) { sc[3] = en_next[e]; return e; }
        return sc[2]++;
    }
    __device__ void free_en(uint32_t e) { en_next[e] = sc[3]; sc[3] = e; }
    __device__ uint32_t alloc_fn(uint32_t freq) {
        uint32_t f = sc[5];
        if (f != LFU_NIL) sc[5] = fn_next[f];
        else f = sc[4]++;
        fn_freq[f] = freq; fn_head[f] = fn_tail[f] = LFU_NIL;
        return f;
    }
    __device__ void append(uint32_t f, uint32_t e) {          // at the most-recent end
        const uint32_t t = fn_tail[f];
        en_prev[e] = t; en_next[e] = LFU_NIL; en_f[e] = f;
        if (t != LFU_NIL) en_next[t] = e; else fn_head[f] = e;
        fn_tail[f] = e;
    }
    __device__ void unlink(uint32_t f, uint32_t e) {
        const uint32_t p = en_prev[e], n = en_next[e];
        if (p != LFU_NIL) en_next[p] = n; else fn_head[f] = n;
        if (n != LFU_NIL) en_prev[n] = p; else fn_tail[f] = p;
    }
    __device__ void fn_insert_after(uint32_t a, uint32_t f) {  // a == NIL: at the front
        const uint32_t n = a == LFU_NIL ? sc[0] : fn_next[a];
        fn_prev[f] = a; fn_next[f] = n;
        if (n != LFU_NIL) fn_prev[n] = f;
        if (a == LFU_NIL) sc[0] = f; else fn_next[a] = f;
    }
    __device__ void fn_remove(uint32_t f) {
        const uint32_t p = fn_prev[f], n = fn_next[f];
        if (p != LFU_NIL) fn_next[p] = n; else sc[0] = n;
        if (n != LFU_NIL) fn_prev[n] = p;
        fn_next[f] = sc[5]; sc[5] = f;
    }
    // get() hit: use count + 1, most recent within its new count (cache.py:91-95)
    __device__ void touch(uint32_t e) {
        const uint32_t f = en_f[e], F = fn_freq[f];
        uint32_t nf = fn_next[f];
        if (nf == LFU_NIL || fn_freq[nf] != F + 1) { nf = alloc_fn(F + 1); fn_insert_after(f, nf); }
        unlink(f, e);
        append(nf, e);
        if (fn_head[f] == LFU_NIL) fn_remove(f);
    }
    // _evict_one (cache.py:117-128): least used, least recently within it
    __device__ void evict() {
        const uint32_t f = sc[0], e = fn_head[f];
        unlink(f, e);
        kc_lfu[en_slot[e]] = LFU_NIL;
        free_en(e);
        sc[1]--;
        if (fn_head[f] == LFU_NIL) fn_remove(f);
    }
    // put() of a fresh key (cache.py:99-109)
    __device__ void insert(uint32_t slot) {
        uint32_t f = sc[0];
        if (f == LFU_NIL || fn_freq[f] != 1) { f = alloc_fn(1); fn_insert_after(LFU_NIL, f); }
        const uint32_t e = alloc_en();
        en_slot[e] = slot;
        append(f, e);
        kc_lfu[slot] = e;
        sc[1]++;
    }
};
}  // namespace lfu

__global__ void k_lfu_reset(DevLfu L, int retain) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= L.S) return;
    unsigned long long *ev = L.ev + (size_t)s * 2;
    ev[1] += ev[0]; ev[0] = 0;
    if (!retain) {
        uint32_t *sc = L.sc + (size_t)s * 8;
        sc[0] = LFU_NIL; sc[1] = 0; sc[2] = 0; sc[3] = LFU_NIL; sc[4] = 0; sc[5] = LFU_NIL;
    }
}

// one thread per stream: replay the logged lookups, fix the window counters;
// hit_out (Table-1 batch API) gets the policy's hit flag of each lookup, the
// stream's lookups starting at hit_base[s]
__global__ void k_lfu_replay(DevStreams S, DevLfu L, uint8_t *hit_out, const uint32_t *hit_base) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S.S || s >= L.S) return;
    const uint32_t n = S.lfu_logn[s];
    lfu::View v(L, s);
    const uint32_t *log = S.lfu_log + (size_t)s * S.lfu_logcap;
    unsigned long long hits = 0, misses = 0, memo_h = 0, memo_m = 0, ev = 0;
    for (uint32_t i = 0; i < n; i++) {
        const uint32_t x = log[i], slot = x & 0x7FFFFFFFu;
        if (x >> 31) memo_m++; else memo_h++;
        const uint32_t e = v.kc_lfu[slot];
        if (hit_out && hit_base[s] != LFU_NIL) hit_out[hit_base[s] + i] = e != LFU_NIL ? 1 : 0;
        if (e != LFU_NIL) { hits++; v.touch(e); continue; }
        misses++;
        if (L.cap == 0) continue;               // capacity below one entry: never stored
        while (v.sc[1] >= L.cap) { v.evict(); ev++; }
        v.insert(slot);
    }
    unsigned long long *st = S.stats + (size_t)s * 8;
    st[1] = st[1] + hits - memo_h;
    st[2] = st[2] + misses - memo_m;
    st[6] = v.sc[1];
    L.ev[(size_t)s * 2] += ev;
    S.lfu_logn[s] = 0;
}

// set_capacity shrink (cache.py:130-137): evict until the resident set fits
__global__ void k_lfu_shrink(DevStreams S, DevLfu L) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= L.S) return;
    lfu::View v(L, s);
    unsigned long long ev = 0;
    while (v.sc[1] > L.cap) { v.evict(); ev++; }
    L.ev[(size_t)s * 2] += ev;
    S.stats[(size_t)s * 8 + 6] = v.sc[1];
}

static int lfu_enqueue(const OtflmStreams *s, cudaStream_t st);
