// tools/research/bestfit_chunk_model.cpp — ANALYSIS PROTOTYPE (not product code): commits per
// speculative chunk of W requests for BEST FIT on config 2 (256 MiB, 4K batches, LU8[16 B, 1 MiB)).
// Speculation = each request takes the smallest piece >= r (lowest address on ties) of the
// chunk-start free set minus the pieces earlier requests of the chunk took (their remainders are
// not visible); the chunk commits up to the first request whose result differs from the
// sequential best fit.
// Build: g++ -O2 -o /tmp/bfm tools/research/bestfit_chunk_model.cpp /tmp/tg.o
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
int main(int argc, char **argv) {
    int nb = argc > 1 ? atoi(argv[1]) : 60;
    const int W = argc > 2 ? atoi(argv[2]) : 32;
    const u64 A = (256ull << 20) / 16, B = 4096, seed = 2405070790ull + 2000;
    tg_t *t = tg_create(0, seed, B, 1, 2, 1000000ull, 0, 4, 20, 0);
    std::vector<u64> fids(B), sz(B), off;
    std::map<u64, u64> fr; fr[0] = A;                 // start -> size
    std::set<std::pair<u64, u64>> bs; bs.insert({A, 0});   // (size, start)
    std::map<u64, u64> live;
    u64 tot_chunks = 0, tot_req = 0;
    for (int b = 0; b < nb; b++) {
        u64 nf, na, fa;
        tg_next_batch(t, B, fids.data(), &nf, sz.data(), &na, &fa);
        std::vector<u64> fo;
        for (u64 j = 0; j < nf; j++) { u64 o = off[fids[j]]; if (o != ~0ull) fo.push_back(o); }
        std::sort(fo.begin(), fo.end());
        for (u64 o : fo) {
            u64 s = live[o]; live.erase(o); u64 st = o, en = o + s;
            auto it = fr.lower_bound(o);
            if (it != fr.end() && it->first == en) { en += it->second; bs.erase({it->second, it->first}); fr.erase(it); }
            it = fr.lower_bound(o);
            if (it != fr.begin()) { auto p = std::prev(it); if (p->first + p->second == st) { st = p->first; bs.erase({p->second, p->first}); fr.erase(p); } }
            fr[st] = en - st; bs.insert({en - st, st});
        }
        std::vector<u64> r(na);
        for (u64 i = 0; i < na; i++) r[i] = (sz[i] + 15) / 16;
        u64 pos = 0, chunks = 0;
        while (pos < na) {
            u64 end = std::min(na, pos + (u64)W);
            chunks++;
            std::set<std::pair<u64, u64>> taken;
            std::vector<u64> spec(end - pos);
            for (u64 i = pos; i < end; i++) {
                auto it = bs.lower_bound({r[i], 0});
                while (it != bs.end() && taken.count(*it)) ++it;
                if (it == bs.end()) { spec[i - pos] = ~0ull; continue; }
                spec[i - pos] = it->second;
                taken.insert(*it);
            }
            u64 i = pos;
            for (; i < end; i++) {
                auto it = bs.lower_bound({r[i], 0});
                u64 tv = it == bs.end() ? ~0ull : it->second;
                if (tv != spec[i - pos] && i > pos) break;
                if (it != bs.end()) {
                    u64 s = it->first, st = it->second;
                    bs.erase(it); fr.erase(st);
                    live[st] = r[i];
                    if (s > r[i]) { fr[st + r[i]] = s - r[i]; bs.insert({s - r[i], st + r[i]}); }
                }
                off.push_back(tv);
            }
            pos = i;
        }
        tot_chunks += chunks; tot_req += na;
        if (b % 10 == 9) printf("batch %d na=%lu F=%zu chunks=%lu commit/chunk=%.2f\n", b, na, fr.size(), chunks, (double)na / chunks);
    }
    printf("W=%d total commit/chunk %.2f\n", W, (double)tot_req / tot_chunks);
}
