// LRU simulation of K2 row-line misses on c4 under several slot visiting orders
// (round 2 design study, profiles/r02_summary.md): gcc -O2 lru_rowsim.c -o lru;
// ./lru <cache MB> <scheme 0 random|1 mode-1|2 mode2xmode3 tiles|3 mode1xmode2|4 serpentine> <b> <c>
// LRU line-cache simulation of K2's A|G row accesses on c4 (3 modes, 128-B lines per row)
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <string.h>
static uint64_t s=88172645463325252ull; static inline uint64_t xr(){s^=s<<13;s^=s>>7;s^=s<<17;return s;}
typedef struct {int64_t prev,next;} N;
int64_t I[3]={4821207,1774269,1805187}; int64_t off[3];
int64_t *where; N* nd; int64_t head=-1,tail=-1,cnt=0,cap; int64_t miss=0;
void touch(int64_t line){ // LRU over line ids
  if(where[line]){ int64_t x=line; // move to head
    if(x!=head){ N*n=&nd[x]; if(n->prev>=0) nd[n->prev].next=n->next; if(n->next>=0) nd[n->next].prev=n->prev; if(tail==x) tail=n->prev;
      n->prev=-1; n->next=head; nd[head].prev=x; head=x; } return; }
  miss++; where[line]=1; nd[line].prev=-1; nd[line].next=head; if(head>=0) nd[head].prev=line; head=line; if(tail<0) tail=line; cnt++;
  if(cnt>cap){ int64_t t=tail; tail=nd[t].prev; nd[tail].next=-1; where[t]=0; cnt--; }
}
typedef struct {uint32_t c[3]; uint32_t key;} S;
int cmp(const void*a,const void*b){uint32_t x=((S*)a)->key,y=((S*)b)->key;return x<y?-1:x>y;}
int main(int argc,char**argv){
  int64_t n=2e7; double mb=atof(argv[1]); int scheme=atoi(argv[2]); int b=atoi(argv[3]), c=atoi(argv[4]);
  off[0]=0; off[1]=I[0]; off[2]=I[0]+I[1]; int64_t L=I[0]+I[1]+I[2];
  where=calloc(L,8); nd=malloc(L*sizeof(N)); cap=(int64_t)(mb*1e6/128);
  S* sm=malloc(n*sizeof(S));
  for(int64_t i=0;i<n;i++){ for(int k=0;k<3;k++) sm[i].c[k]=xr()%I[k];
    if(scheme==0) sm[i].key=0;
    else if(scheme==1) sm[i].key=(uint32_t)((uint64_t)sm[i].c[0]*32768/I[0]);
    else if(scheme==2) { uint32_t bb=(uint64_t)sm[i].c[1]*b/I[1], cc=(uint64_t)sm[i].c[2]*c/I[2]; sm[i].key=bb*c+cc; }
    else if(scheme==3) { uint32_t aa=(uint64_t)sm[i].c[0]*b/I[0], bb=(uint64_t)sm[i].c[1]*c/I[1]; sm[i].key=aa*c+bb; }
    else if(scheme==4) { uint32_t bb=(uint64_t)sm[i].c[1]*b/I[1], cc=(uint64_t)sm[i].c[2]*c/I[2]; if(bb&1) cc=c-1-cc; sm[i].key=bb*c+cc; } // serpentine
  }
  if(scheme) qsort(sm,n,sizeof(S),cmp);
  for(int it=0;it<2;it++){ miss=0; for(int64_t i=0;i<n;i++) for(int k=0;k<3;k++) touch(off[k]+sm[i].c[k]); }
  printf("cache %.0fMB scheme %d b=%d c=%d: misses/iter %.2fM (%.2f per sample)\n",mb,scheme,b,c,miss/1e6,(double)miss/n);
}
