// tools/research/tlsf_window_fixpoint.cpp — ANALYSIS PROTOTYPE (not product code, not used by tests
// or bench.py): measures how an exact parallel formulation of the TLSF alloc phase would converge.
//
// The alloc phase of one config-3/5 batch is replayed sequentially (the exact answer), then again
// window by window (W consecutive requests from the exact window-start state): each iteration
// "sweeps" the classes bottom-up — class k serves its demand stream (its own requests plus those
// passed up from class k-1, in time order) from its members (batch-start pieces plus the remainder
// ARRIVALS guessed by the previous iteration, each present from its creation time), lowest address
// first, with head carves staying in the class — and recomputes the arrivals; a window is done when
// the arrivals are a fixpoint.  Every window's result is checked against the sequential answer.
// Build: gcc -O2 -c tracegen/tracegen.c -o /tmp/tg.o && g++ -O2 -std=c++17 -o /tmp/fx
//        tools/research/tlsf_window_fixpoint.cpp /tmp/tg.o && /tmp/fx <cfg 3|5> <batch> <W>
// Results: config 3 batch 20, W = 256 / 1024 / 4096: 3.7 / 6.9 / 18.6 sweeps per
// window on average, most windows 2-3, a few 10-112 (descending carve chains).  Config 5 batch 4,
// W = 1024: 53 sweeps per window on average (max 525; 145 of 615 windows need >= 11); W = 4096: a
// window does not reach a fixpoint within 1000 sweeps (the iteration oscillates) -> reported as a
// mismatch.  Plain Jacobi over whole assignments fixes only ~128 requests per iteration.
// Class-sweep fixpoint for exact TLSF alloc batches (research prototype): iterate on the set of
// remainder arrivals; each iteration sweeps classes bottom-up with known arrivals.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <set>
#include <map>
#include <queue>
#include <vector>
#include <algorithm>
extern "C" {
typedef struct tg tg_t;
tg_t *tg_create(int, uint64_t, uint64_t, uint64_t, uint64_t, uint64_t, int, uint64_t, uint64_t, uint64_t);
int tg_next_batch(tg_t *t, uint64_t max_n, uint64_t *free_ids, uint64_t *nf_out, uint64_t *sizes, uint64_t *na_out, uint64_t *first);
}
static int flog2(uint64_t u){return 63-__builtin_clzll(u);}
static uint64_t icls(uint64_t u){ const int L=5; if(u<(1ull<<L))return u; int m=flog2(u); return (uint64_t)(m-L+1)*(1ull<<L)+((u>>(m-L))-(1ull<<L));}
static uint64_t scls(uint64_t u){ const int L=5; if(u<(1ull<<L))return icls(u); int m=flog2(u); return icls(u+(1ull<<(m-L))-1);}
static uint64_t lo_of(uint64_t c){ const int L=5; uint64_t fl=c>>L, sl=c&31; return fl==0? sl : ((32+sl)<<(fl-1)); }
struct Arr { long t; long f; uint64_t R; };   // after request t, piece f has R units (class icls(R))
int main(int argc,char**argv){
  int cfg=argc>1?atoi(argv[1]):3; int target=argc>2?atoi(argv[2]):20;
  uint64_t A,B,seed; if(cfg==5){A=1ull<<32;B=1<<20;seed=2405070790ull+5000;} else {A=(4ull<<30)/16;B=65536;seed=2405070790ull+3000;}
  tg_t*t=tg_create(0,seed,B,2,5,100000000ull,0,4,12,0);
  std::vector<uint64_t> fids(B),sz(B),off;
  std::map<uint64_t,uint64_t> fr; fr[0]=A; std::map<uint64_t,uint64_t> live;
  std::set<std::pair<uint64_t,uint64_t>> cs; cs.insert({icls(A),0});
  for(int b=0;b<=target;b++){
    uint64_t nf,na,fa; tg_next_batch(t,B,fids.data(),&nf,sz.data(),&na,&fa);
    std::vector<uint64_t> fo; for(uint64_t j=0;j<nf;j++){uint64_t o=off[fids[j]]; if(o!=~0ull) fo.push_back(o);}
    std::sort(fo.begin(),fo.end());
    for(uint64_t o:fo){ uint64_t s=live[o]; live.erase(o); uint64_t st=o,en=o+s;
      auto it=fr.lower_bound(o); if(it!=fr.end()&&it->first==en){en+=it->second; cs.erase({icls(it->second),it->first}); fr.erase(it);}
      it=fr.lower_bound(o); if(it!=fr.begin()){auto p=std::prev(it); if(p->first+p->second==st){st=p->first; cs.erase({icls(p->second),p->first}); fr.erase(p);}}
      fr[st]=en-st; cs.insert({icls(en-st),st}); }
    if(b==target){
      std::vector<uint64_t> pz; for(auto&kv:fr) pz.push_back(kv.second);
      size_t F=pz.size(); std::vector<uint64_t> r(na), c(na);
      for(uint64_t i=0;i<na;i++){ r[i]=(sz[i]+15)/16; c[i]=scls(r[i]); }
      std::vector<long> exact(na,-1);
      { std::vector<uint64_t> R=pz; std::set<std::pair<uint64_t,long>> S; for(size_t f=0;f<F;f++) S.insert({icls(R[f]),(long)f});
        for(uint64_t i=0;i<na;i++){ auto it=S.lower_bound({c[i],-1}); if(it==S.end()) continue; long f=it->second; S.erase(it); exact[i]=f; R[f]-=r[i]; if(R[f]) S.insert({icls(R[f]),f}); } }
      uint64_t KMAX=icls(A)+1;
      long W = argc>3? atol(argv[3]) : 2048;
      std::vector<uint64_t> Rst=pz;          // exact state at window start
      long tot_it=0, nwin=0, maxit=0; std::vector<int> hist(12,0);
      for(long w0=0; w0<(long)na; w0+=W){
        long w1=std::min((long)na,w0+W); nwin++;
        std::vector<std::vector<long>> base(KMAX+1);
        for(size_t f=0;f<F;f++) if(Rst[f]) base[icls(Rst[f])].push_back((long)f);
        std::vector<Arr> arr; std::vector<long> ch;
        int it;
        for(it=0; it<1000; it++){
          std::vector<std::vector<Arr>> ain(KMAX+1); for(auto&a:arr) ain[icls(a.R)].push_back(a);
          for(auto&v:ain) std::sort(v.begin(),v.end(),[](const Arr&x,const Arr&y){return x.t<y.t;});
          std::vector<Arr> narr; std::vector<long> nch(w1-w0,-1);
          std::vector<long> up;
          std::vector<std::vector<long>> own(KMAX+1); for(long i=w0;i<w1;i++) own[c[i]].push_back(i);
          for(uint64_t k=0;k<=KMAX;k++){
            if(own[k].empty() && up.empty()) continue;
            std::vector<long> D; std::merge(own[k].begin(),own[k].end(),up.begin(),up.end(),std::back_inserter(D));
            std::vector<long> nup;
            std::priority_queue<std::pair<long,uint64_t>,std::vector<std::pair<long,uint64_t>>,std::greater<>> pq;
            for(long f: base[k]) pq.push({f,Rst[f]});
            size_t ai=0; auto &AV=ain[k];
            for(long i: D){
              while(ai<AV.size() && AV[ai].t < i){ pq.push({AV[ai].f, AV[ai].R}); ai++; }
              if(pq.empty()){ nup.push_back(i); continue; }
              auto top=pq.top(); pq.pop(); long f=top.first; uint64_t R=top.second;
              nch[i-w0]=f; R-=r[i];
              if(R && icls(R)==k) pq.push({f,R});
              else narr.push_back({i,f,R});
            }
            up.swap(nup);
          }
          bool same = narr.size()==arr.size();
          if(same){ std::vector<std::tuple<long,long,uint64_t>> a1,a2; for(auto&x:arr) a1.push_back({x.t,x.f,x.R}); for(auto&x:narr) a2.push_back({x.t,x.f,x.R}); std::sort(a1.begin(),a1.end()); std::sort(a2.begin(),a2.end()); same = a1==a2; }
          arr.swap(narr); ch.swap(nch);
          if(same) break;
        }
        // verify and apply
        for(long i=w0;i<w1;i++){ if(ch[i-w0]!=exact[i]){ printf("MISMATCH window %ld at %ld\n", w0, i); return 1; } }
        for(long i=w0;i<w1;i++){ long f=ch[i-w0]; if(f>=0) Rst[f]-=r[i]; }
        tot_it+=it+1; maxit=std::max(maxit,(long)it+1); hist[std::min(it+1,11)]++;
      }
      printf("W=%ld windows %ld, sweeps total %ld (avg %.2f, max %ld)  hist:", W, nwin, tot_it, double(tot_it)/nwin, maxit);
      for(int h=1;h<12;h++) printf(" %d:%d",h,hist[h]); printf("\n");
    }
    for(uint64_t i=0;i<na;i++){ uint64_t rr=(sz[i]+15)/16; auto it=cs.lower_bound({scls(rr),0}); if(it==cs.end()){off.push_back(~0ull);continue;}
      uint64_t st=it->second,s=fr[st]; cs.erase(it); fr.erase(st); off.push_back(st); live[st]=rr; if(s>rr){fr[st+rr]=s-rr; cs.insert({icls(s-rr),st+rr});} }
  }
}
