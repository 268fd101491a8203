// Exhaustive check of the device draw's r % b (lp_device.cuh mod64_small): every b < 2^16,
// 2000 random 64-bit r each plus edge values, against the 64-bit % operator.
//   gcc -O2 -o barrett_check barrett_check.c && ./barrett_check   -> bad=0
#include <stdio.h>
#include <stdint.h>
static uint64_t s=0x12345;
static uint64_t rnd(){ s+=0x9e3779b97f4a7c15ULL; uint64_t z=s; z=(z^(z>>30))*0xbf58476d1ce4e5b9ULL; z=(z^(z>>27))*0x94d049bb133111ebULL; return z^(z>>31);}
static uint32_t bmod(uint32_t a, uint32_t m, uint32_t d){ uint32_t q=(uint32_t)(((uint64_t)a*m)>>32); uint32_t r=a-q*d; return r>=d? r-d : r; }
int main(){
  long bad=0;
  for(uint32_t d=1; d<=65535; ++d){
    uint32_t m = d==1 ? 0xffffffffu : (uint32_t)((1ull<<32)/d);
    uint32_t c32=(uint32_t)((1ull<<32)%d);
    for(int t=0;t<2000;++t){
      uint64_t r=rnd(); if(t<4) r = t==0?0: t==1? ~0ull : t==2? ((uint64_t)d<<32)-1 : (uint64_t)-1 - d;
      uint32_t h=bmod((uint32_t)(r>>32),m,d), l=bmod((uint32_t)r,m,d);
      uint32_t x=h*c32+l; uint32_t got=bmod(x,m,d);
      if(got!=r%d){ if(bad<5) printf("bad d=%u r=%llu got %u want %llu\n",d,(unsigned long long)r,got,(unsigned long long)(r%d)); ++bad;}
    }
  }
  printf("bad=%ld\n",bad); return 0;}
