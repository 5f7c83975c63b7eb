// tools/research/chunk_commit_model.cpp — ANALYSIS PROTOTYPE (not product code, not used by tests
// or bench.py): how many requests a speculative chunk of W candidates commits on config 5.
// Model: a chunk speculates every candidate against the chunk-start state with the remainders that
// CHANGE class dropped (a carve that stays in its class is kept — a head carve); it commits up to
// the first candidate whose speculative result differs from the sequential one.  Requests whose
// search class is above the highest non-wilderness class at chunk start are WILD and never enter a
// chunk (the wilderness split).  Prints commits per chunk for W = 32, 64, 128 on the same batches
// (the true state always advances by the sequential replay).
// Build: gcc -O2 -c tracegen/tracegen.c -o /tmp/tg.o && g++ -O2 -o /tmp/ccm tools/research/chunk_commit_model.cpp /tmp/tg.o
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <set>
#include <map>
#include <vector>
#include <algorithm>
extern "C" {
typedef struct tg tg_t;
tg_t *tg_create(int model, uint64_t seed, uint64_t batch, uint64_t rho_num, uint64_t rho_den,
                uint64_t total_ops, int size_kind, uint64_t a, uint64_t b, uint64_t n_slots);
int tg_next_batch(tg_t *t, uint64_t max_n, uint64_t *free_ids, uint64_t *nf_out,
                  uint64_t *sizes, uint64_t *na_out, uint64_t *first_alloc_id);
}
typedef uint64_t u64;
static int flog2(u64 u) { return 63 - __builtin_clzll(u); }
static u64 icls(u64 u, int L = 5) {
    if (u < (1ull << L)) return u;
    int m = flog2(u);
    return (u64)(m - L + 1) * (1ull << L) + ((u >> (m - L)) - (1ull << L));
}
static u64 scls(u64 u, int L = 5) {
    if (u < (1ull << L)) return icls(u);
    int m = flog2(u);
    return icls(u + (1ull << (m - L)) - 1);
}
typedef std::set<std::pair<u64, u64>> CS;   // (class, start)

int main(int argc, char **argv) {
    int nb = argc > 1 ? atoi(argv[1]) : 8;
    int first_b = argc > 2 ? atoi(argv[2]) : 1;
    const int FIX = argc > 3 ? atoi(argv[3]) : 0;   // mismatching requests a chunk may fix in place
    const u64 A = 1ull << 32, B = 1 << 20, seed = 2405070790ull + 5000;
    tg_t *t = tg_create(0, seed, B, 2, 5, 100000000ull, 0, 4, 12, 0);
    std::vector<u64> fids(B), sz(B), off;
    std::map<u64, u64> fr;
    fr[0] = A;
    CS cs;
    cs.insert({icls(A), 0});
    std::map<u64, u64> live;
    const int NW = 3;
    const int Ws[NW] = {32, 64, 128};
    for (int b = 0; b < nb; b++) {
        u64 nf, na, fa;
        tg_next_batch(t, B, fids.data(), &nf, sz.data(), &na, &fa);
        std::vector<u64> fo;
        for (u64 j = 0; j < nf; j++) { u64 o = off[fids[j]]; if (o != ~0ull) fo.push_back(o); }
        std::sort(fo.begin(), fo.end());
        for (u64 o : fo) {
            u64 s = live[o]; live.erase(o); u64 st = o, en = o + s;
            auto it = fr.lower_bound(o);
            if (it != fr.end() && it->first == en) { en += it->second; cs.erase({icls(it->second), it->first}); fr.erase(it); }
            it = fr.lower_bound(o);
            if (it != fr.begin()) { auto p = std::prev(it); if (p->first + p->second == st) { st = p->first; cs.erase({icls(p->second), p->first}); fr.erase(p); } }
            fr[st] = en - st; cs.insert({icls(en - st), st});
        }
        std::vector<u64> r(na), c(na);
        for (u64 i = 0; i < na; i++) { r[i] = (sz[i] + 15) / 16; c[i] = scls(r[i]); }
        // wilderness: the highest piece (the arena's tail) — removed from the class state
        auto wl = std::prev(cs.end());
        u64 wst = wl->second, wsz = fr[wst];
        bool do_model = b >= first_b;
        if (do_model) { cs.erase(wl); fr.erase(wst); }
        // the models run on copies of the batch-start state (W loop), the real replay last
        std::vector<u64> res(na);
        for (int wi = 0; wi < (do_model ? NW : 0) + 1; wi++) {
            const bool model = wi < NW && do_model;
            const int W = model ? Ws[wi] : 0;
            CS C = cs;
            std::map<u64, u64> Fr = fr;
            u64 chunks = 0, committed = 0, wildn = 0, full = 0;
            u64 pos = 0;
            std::vector<u64> cand;
            std::vector<u64> spec;
            while (pos < na) {
                if (!model) {   // plain sequential replay (results into res)
                    u64 i = pos++;
                    auto it = C.lower_bound({c[i], 0});
                    if (it == C.end()) { res[i] = ~1ull; continue; }
                    u64 k = it->first, st = it->second, s = Fr[st];
                    C.erase(it); Fr.erase(st);
                    res[i] = st;
                    if (s > r[i]) { Fr[st + r[i]] = s - r[i]; C.insert({icls(s - r[i]), st + r[i]}); }
                    (void)k;
                    continue;
                }
                // candidates: next W requests with search class <= highest class now
                u64 Mx = C.empty() ? 0 : std::prev(C.end())->first;
                cand.clear();
                u64 q = pos;
                while (cand.size() < (size_t)W && q < na) {
                    if (!C.empty() && c[q] <= Mx) cand.push_back(q);
                    else wildn++;
                    q++;
                }
                if (cand.empty()) { pos = q; continue; }
                chunks++;
                // speculative replay: overlay of removed pieces and in-class carves
                std::map<u64, u64> carved;     // start(batch key) -> current start
                std::set<std::pair<u64, u64>> removed;
                spec.assign(cand.size(), 0);
                for (size_t j = 0; j < cand.size(); j++) {
                    u64 i = cand[j];
                    auto it = C.lower_bound({c[i], 0});
                    while (it != C.end() && removed.count(*it)) ++it;
                    if (it == C.end()) { spec[j] = ~1ull; continue; }
                    u64 key = it->second;
                    u64 cur = carved.count(key) ? carved[key] : key;
                    u64 end = key + Fr[key];
                    spec[j] = cur;
                    u64 ns = cur + r[i];
                    if (end > ns && icls(end - ns) == it->first) carved[key] = ns;
                    else removed.insert(*it);
                }
                // true replay, stop at the first mismatch (FIX > 0: at the (FIX+1)-th; an upper
                // bound for fixing a dirty request in place when the later ones stay valid)
                size_t j = 0;
                int fixes = 0;
                for (; j < cand.size(); j++) {
                    u64 i = cand[j];
                    auto it = C.lower_bound({c[i], 0});
                    u64 tv = it == C.end() ? ~1ull : it->second;
                    if (tv != spec[j] && j > 0 && fixes++ >= FIX) break;
                    if (it != C.end()) {
                        u64 st = it->second, s = Fr[st];
                        C.erase(it); Fr.erase(st);
                        if (s > r[i]) { Fr[st + r[i]] = s - r[i]; C.insert({icls(s - r[i]), st + r[i]}); }
                    }
                }
                committed += j;
                if (j == cand.size()) { full++; pos = q; }
                else pos = cand[j];
                // requests skipped as WILD before cand[j] are counted again if re-scanned; fine
            }
            if (model)
                printf("batch %d W=%d chunks=%lu commit/chunk=%.2f full=%.3f\n", b, W, chunks,
                       (double)committed / chunks, (double)full / chunks);
            else {
                // commit the batch: results, live map; wilderness serves the WILD ones in order
                for (u64 i = 0; i < na; i++) {
                    if (res[i] == ~1ull) {
                        if (do_model) { res[i] = wst; wst += r[i]; wsz -= r[i]; }
                        else res[i] = ~0ull;
                    }
                    off.push_back(res[i]);
                    if (res[i] != ~0ull) live[res[i]] = r[i];
                }
                cs = C; fr = Fr;
                if (do_model) { fr[wst] = wsz; cs.insert({icls(wsz), wst}); }
            }
        }
        fflush(stdout);
    }
}
