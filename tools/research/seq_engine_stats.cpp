// tools/research/seq_engine_stats.cpp — ANALYSIS PROTOTYPE (not product code, not used by tests or
// bench.py): statistics of the strictly sequential TLSF alloc phase that decide the data layout of
// a one-thread engine — how many remainders arrive per batch, how many are alive at once (could the
// arrival sets live in shared memory?), how often consecutive requests touch the same class.
// Build: g++ -O2 -o /tmp/ses tools/research/seq_engine_stats.cpp tracegen/tracegen.c
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
static int flog2(uint64_t u) { return 63 - __builtin_clzll(u); }
static uint64_t icls(uint64_t u, int L = 5) {
    if (u < (1ull << L)) return u;
    int m = flog2(u);
    return (uint64_t)(m - L + 1) * (1ull << L) + ((u >> (m - L)) - (1ull << L));
}
static uint64_t scls(uint64_t u, int L = 5) {
    if (u < (1ull << L)) return icls(u);
    int m = flog2(u);
    return icls(u + (1ull << (m - L)) - 1);
}
int main(int argc, char **argv) {
    int cfg = argc > 1 ? atoi(argv[1]) : 5;
    int nb = argc > 2 ? atoi(argv[2]) : 8;
    int H = argc > 3 ? atoi(argv[3]) : 8;
    uint64_t A, B;
    uint64_t seed;
    if (cfg == 5) { A = 1ull << 32; B = 1 << 20; seed = 2405070790ull + 5000; }
    else { A = (4ull << 30) / 16; B = 65536; seed = 2405070790ull + 3000; }
    tg_t *t = tg_create(0, seed, B, 2, 5, 100000000ull, 0, 4, 12, 0);
    std::vector<uint64_t> fids(B), sz(B), off;
    std::map<uint64_t, uint64_t> fr; fr[0] = A;
    std::set<std::pair<uint64_t, uint64_t>> cs; cs.insert({icls(A), 0});
    std::map<uint64_t, uint64_t> live;
    for (int b = 0; b < nb; b++) {
        uint64_t nf, na, fa;
        tg_next_batch(t, B, fids.data(), &nf, sz.data(), &na, &fa);
        std::vector<uint64_t> fo;
        for (uint64_t j = 0; j < nf; j++) { uint64_t o = off[fids[j]]; if (o != ~0ull) fo.push_back(o); }
        std::sort(fo.begin(), fo.end());
        for (uint64_t o : fo) {
            uint64_t s = live[o]; live.erase(o); uint64_t st = o, en = o + s;
            auto it = fr.lower_bound(o);
            if (it != fr.end() && it->first == en) { en += it->second; cs.erase({icls(it->second), it->first}); fr.erase(it); }
            it = fr.lower_bound(o);
            if (it != fr.begin()) { auto p = std::prev(it); if (p->first + p->second == st) { st = p->first; cs.erase({icls(p->second), p->first}); fr.erase(p); } }
            fr[st] = en - st; cs.insert({icls(en - st), st});
        }
        uint64_t F = fr.size();
        // batch-start membership: a piece is "csr" while it is still its batch-start block in
        // its batch-start class; an arrival otherwise
        std::set<uint64_t> bs_key;            // starts of batch-start blocks not yet touched
        for (auto &kv : fr) bs_key.insert(kv.first);
        std::map<uint64_t, int> ncls;          // members per class now
        for (auto &e : cs) ncls[e.first]++;
        std::set<std::pair<uint64_t, uint64_t>> arr;   // alive arrivals (class, start)
        long arrivals = 0, peak_arr = 0, head_is_arr = 0, pops = 0, same_prev_k = 0, k_eq_prev_nk = 0;
        long first_ge_changed = 0, overflowed = 0, peak_over = 0, nonempty_peak = 0;
        uint64_t pk = ~0ull, pnk = ~0ull;
        std::map<uint64_t, std::set<uint64_t>> cls_members;   // for "beyond the H smallest"
        for (auto &e : cs) cls_members[e.first].insert(e.second);
        long beyond = 0;   // arrivals that land beyond the H smallest of their class
        for (uint64_t i = 0; i < na; i++) {
            uint64_t r = (sz[i] + 15) / 16; uint64_t c = scls(r);
            auto it = cs.lower_bound({c, 0});
            if (it == cs.end()) { off.push_back(~0ull); continue; }
            uint64_t k = it->first, st = it->second, s = fr[st];
            if (k == pk) same_prev_k++;
            if (k == pnk) k_eq_prev_nk++;
            bool isarr = arr.count({k, st});
            if (isarr) head_is_arr++;
            cs.erase(it); fr.erase(st); off.push_back(st); live[st] = r;
            cls_members[k].erase(st);
            uint64_t nk = ~0ull;
            if (s > r) {
                uint64_t ns = st + r, nsz = s - r; nk = icls(nsz);
                fr[ns] = nsz; cs.insert({nk, ns});
                if (nk != k) {
                    arrivals++;
                    if (isarr) arr.erase({k, st});
                    arr.insert({nk, ns});
                    auto &m = cls_members[nk];
                    m.insert(ns);
                    long rank = 0;
                    for (auto q = m.begin(); q != m.end() && *q != ns && rank < H; ++q) rank++;
                    if (rank >= H) beyond++;
                } else {
                    if (isarr) { arr.erase({k, st}); arr.insert({k, ns}); }
                    cls_members[k].insert(ns);
                }
            } else if (isarr) arr.erase({k, st});
            if (nk != k) pops++;
            peak_arr = std::max(peak_arr, (long)arr.size());
            pk = k; pnk = nk;
        }
        printf("batch %d nf=%lu na=%lu F=%lu arrivals=%ld peak_alive_arrivals=%ld head_is_arrival=%ld pops=%ld "
               "k==prev_k %.3f k==prev_nk %.3f beyondH=%ld live=%zu\n",
               b, nf, na, F, arrivals, peak_arr, head_is_arr, pops, (double)same_prev_k / na,
               (double)k_eq_prev_nk / na, beyond, live.size());
        fflush(stdout);
    }
}
