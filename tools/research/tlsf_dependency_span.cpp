// tools/research/tlsf_dependency_span.cpp — ANALYSIS PROTOTYPE (not product code, not used by tests
// or bench.py): the critical path of a TLSF alloc batch under a simple dependency model.  Request i
// depends on the request that created the remainder it takes (if it changed class) and on the last
// request that emptied, refilled or re-headed any class in [c_i, k_i) — rank-matched pops inside a
// class and head carves in place are not dependencies.  Config 5, batches 1-4: span 66k, 49k, 39k,
// 33k steps for 629k requests (average parallelism 10-19); see DESIGN.md §12.
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
static int flog2(uint64_t u){return 63-__builtin_clzll(u);}
static uint64_t icls(uint64_t u,int L=5){ if(u<(1ull<<L))return u; int m=flog2(u); return (uint64_t)(m-L+1)*(1ull<<L)+((u>>(m-L))-(1ull<<L));}
static uint64_t scls(uint64_t u,int L=5){ if(u<(1ull<<L))return icls(u); int m=flog2(u); return icls(u+(1ull<<(m-L))-1);}
int main(int argc,char**argv){
  int cfg=argc>1?atoi(argv[1]):5; int nb=argc>2?atoi(argv[2]):8;
  uint64_t A,B; int rn=2,rd=5; uint64_t seed;
  if(cfg==5){A=1ull<<32;B=1<<20;seed=2405070790ull+5000;} else {A=(4ull<<30)/16;B=65536;seed=2405070790ull+3000;}
  tg_t*t=tg_create(0,seed,B,rn,rd,100000000ull,0,4,12,0);
  std::vector<uint64_t> fids(B),sz(B),off; // id->offset
  std::map<uint64_t,uint64_t> fr; fr[0]=A; // start->size
  std::set<std::pair<uint64_t,uint64_t>> cs; cs.insert({icls(A),0});
  std::map<uint64_t,uint64_t> live;
  for(int b=0;b<nb;b++){
    uint64_t nf,na,fa; tg_next_batch(t,B,fids.data(),&nf,sz.data(),&na,&fa);
    std::vector<uint64_t> fo; for(uint64_t j=0;j<nf;j++){uint64_t o=off[fids[j]]; if(o!=~0ull) fo.push_back(o);}
    std::sort(fo.begin(),fo.end());
    for(uint64_t o:fo){ uint64_t s=live[o]; live.erase(o); uint64_t st=o,en=o+s;
      auto it=fr.lower_bound(o); if(it!=fr.end()&&it->first==en){en+=it->second; cs.erase({icls(it->second),it->first}); fr.erase(it);} 
      it=fr.lower_bound(o); if(it!=fr.begin()){auto p=std::prev(it); if(p->first+p->second==st){st=p->first; cs.erase({icls(p->second),p->first}); fr.erase(p);}}
      fr[st]=en-st; cs.insert({icls(en-st),st}); }
    // stats on batch start
    uint64_t F=fr.size();
    std::map<uint64_t,int> bsblk; for(auto&kv:fr) bsblk[kv.first]=1;
    uint64_t exact=0,spill=0,wild=0,fromRem=0,drops=0,dropsLow=0; uint64_t maxc=0;
    std::vector<long> remby; std::map<uint64_t,long> creator; // block start->request that created it as remainder
    std::vector<int> depth(na,0); long gh[5]={0,0,0,0,0}; std::vector<int> ld(2048,0); int span=0; std::map<uint64_t,int> bd; std::vector<int> cnt(2048,0); for(auto&e:cs) if(e.first<2048) cnt[e.first]++; int maxd=0; long sumgap=0;
    uint64_t top= A; // wilderness detection: class >= icls(2^20)
    for(uint64_t i=0;i<na;i++){
      uint64_t r=(sz[i]+15)/16; uint64_t c=scls(r); maxc=std::max(maxc,c);
      auto it=cs.lower_bound({c,0}); if(it==cs.end()){off.push_back(~0ull);continue;}
      uint64_t k=it->first, st=it->second, s=fr[st]; int dp=0; for(uint64_t q=c;q<k && q<2048;q++) dp=std::max(dp,ld[q]); {auto b=bd.find(st); if(b!=bd.end()){dp=std::max(dp,b->second); bd.erase(b);}} 
      if(k==c) exact++; else spill++;
      if(k>=icls(1<<20)) wild++;
      auto cr=creator.find(st); int d=0; if(cr!=creator.end()){fromRem++; d=depth[cr->second]+1; long g=i-cr->second; sumgap+=g; int bk=g<=1?0:g<=32?1:g<=1024?2:g<=32768?3:4; gh[bk]++; creator.erase(cr);} depth[i]=d; maxd=std::max(maxd,d);
      cs.erase(it); fr.erase(st); off.push_back(st); live[st]=r;
      int nd=dp+1; span=std::max(span,nd); uint64_t nk0= s>r? icls(s-r):~0ull; if(nk0!=k && k<2048){ cnt[k]--; if(cnt[k]==0) ld[k]=std::max(ld[k],nd);} if(s>r){ uint64_t ns=st+r, nsz=s-r; fr[ns]=nsz; uint64_t nk=icls(nsz); if(nk!=k){ bd[ns]=nd; if(nk<2048){ auto h=cs.lower_bound({nk,0}); bool newhead = (h==cs.end()||h->first!=nk|| h->second>ns); cnt[nk]++; if(newhead) ld[nk]=std::max(ld[nk],nd);} } else bd[ns]=dp; cs.insert({nk,ns}); creator[ns]=i; if(nk!=k){drops++; if(nk<160) dropsLow++;} }
    }
    printf("batch %d nf=%lu na=%lu F=%lu exact=%lu spill=%lu wild=%lu fromRem=%lu drops=%lu dropsLow=%lu maxdepth=%d maxc=%lu avggap=%.1f live=%zu\n",b,nf,na,F,exact,spill,wild,fromRem,drops,dropsLow,maxd,maxc,fromRem?double(sumgap)/fromRem:0.0,live.size()); printf("  span=%d ",span); printf("  gaps <=1 %ld <=32 %ld <=1K %ld <=32K %ld more %ld\n",gh[0],gh[1],gh[2],gh[3],gh[4]);
  }
}
