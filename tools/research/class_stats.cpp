// per-class statistics of a config-5 batch under the sequential replay (analysis only)
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
static u64 icls(u64 u, int L = 5) { if (u < (1ull << L)) return u; int m = flog2(u); return (u64)(m - L + 1) * (1ull << L) + ((u >> (m - L)) - (1ull << L)); }
static u64 scls(u64 u, int L = 5) { if (u < (1ull << L)) return icls(u); int m = flog2(u); return icls(u + (1ull << (m - L)) - 1); }
int main(int argc, char **argv) {
    int nb = atoi(argv[1]); int H = atoi(argv[2]);
    const u64 A = 1ull << 32, B = 1 << 20, seed = 2405070790ull + 5000;
    tg_t *t = tg_create(0, seed, B, 2, 5, 100000000ull, 0, 4, 12, 0);
    std::vector<u64> fids(B), sz(B), off;
    std::map<u64, u64> fr; fr[0] = A;
    std::set<std::pair<u64,u64>> cs; cs.insert({icls(A), 0});
    std::map<u64, u64> live;
    for (int b = 0; b < nb; b++) {
        u64 nf, na, fa; tg_next_batch(t, B, fids.data(), &nf, sz.data(), &na, &fa);
        std::vector<u64> fo;
        for (u64 j = 0; j < nf; j++) { u64 o = off[fids[j]]; if (o != ~0ull) fo.push_back(o); }
        std::sort(fo.begin(), fo.end());
        for (u64 o : fo) { u64 s = live[o]; live.erase(o); u64 st = o, en = o + s;
            auto it = fr.lower_bound(o);
            if (it != fr.end() && it->first == en) { en += it->second; cs.erase({icls(it->second), it->first}); fr.erase(it); }
            it = fr.lower_bound(o);
            if (it != fr.begin()) { auto p = std::prev(it); if (p->first + p->second == st) { st = p->first; cs.erase({icls(p->second), p->first}); fr.erase(p); } }
            fr[st] = en - st; cs.insert({icls(en - st), st}); }
        bool rep = b == nb - 1;
        std::map<u64, long> init, pops, arrs, over, maxover, carves, maxcnt;
        std::map<u64, std::set<u64>> batchset;   // class -> batch-start members still untouched (by start)
        std::map<u64, std::set<u64>> ovset;      // class -> overflow members (start)
        std::map<u64, std::set<u64>> members;    // class -> all members
        if (rep) for (auto &e : cs) { init[e.first]++; members[e.first].insert(e.second); }
        u64 maxk = 0; for (auto &e : cs) maxk = std::max(maxk, e.first);
        for (u64 i = 0; i < na; i++) {
            u64 r = (sz[i] + 15) / 16, c = scls(r);
            auto it = cs.lower_bound({c, 0});
            if (it == cs.end()) { off.push_back(~0ull); continue; }
            u64 k = it->first, st = it->second, s = fr[st];
            cs.erase(it); fr.erase(st); off.push_back(st); live[st] = r;
            if (rep) members[k].erase(st);
            if (s > r) { u64 nk = icls(s - r); fr[st + r] = s - r; cs.insert({nk, st + r});
                if (rep) { members[nk].insert(st + r);
                    if (nk != k) { pops[k]++; arrs[nk]++;
                        // rank of the arrival among members
                        auto &m = members[nk]; long rk = std::distance(m.begin(), m.find(st + r));
                        if (rk >= H) over[nk]++; }
                    else carves[k]++; } }
            else if (rep) pops[k]++;
            if (rep) maxcnt[k] = std::max(maxcnt[k], (long)members[k].size());
        }
        if (rep) {
            printf("batch %d F=%zu maxclass_at_start=%lu\n", b, fr.size(), maxk);
            long tot_over = 0, ncls = 0;
            for (u64 k = 0; k < 1000; k++) {
                if (!init[k] && !pops[k] && !arrs[k]) continue;
                ncls++; tot_over += over[k];
                printf("k=%3lu lo=%6lu init=%6ld pops=%6ld arr=%6ld over=%6ld carves=%6ld maxcnt=%6ld\n", k,
                       (u64)(k < 32 ? k : ((32 + (k & 31)) << ((k >> 5) - 1))), init[k], pops[k], arrs[k], over[k], carves[k], maxcnt[k]);
            }
            printf("classes=%ld over_total=%ld\n", ncls, tot_over);
        }
    }
}
