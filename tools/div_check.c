// Diagnostics: the LL FP8 quantiser divides x / scale as q = x * rcp(d) plus one
// FMA residual correction (csrc/ll.cu wire_chunk).  This checks that sequence
// against IEEE single-precision division on ~10^9 random (x, d) pairs in the
// range the kernel uses it for.   gcc -O2 -ffp-contract=off tools/div_check.c -lm
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
static uint64_t s=88172645463325252ull; static uint32_t nx(){ s^=s<<13; s^=s>>7; s^=s<<17; return (uint32_t)s;}
static float fu(uint32_t u){ float f; memcpy(&f,&u,4); return f;}
int main(){
  long bad=0,n=0;
  for(long it=0; it<1500000000L; ++it){
    float amax = fu((nx() % (uint32_t)(230u<<23)) + (20u<<23));
    float d = amax/448.0f;
    if (d < 0x1p-100f || d > 0x1p100f) continue;
    float x; uint32_t m=nx()%4;
    if(m==0) x=amax; else if(m==1) x=-amax*(float)(nx()%100000)/100000.0f; else if (m==2) x=fu(nx()); else x = fu((nx()&0x807FFFFF)|((uint32_t)((nx()%40)+ ((*(uint32_t*)&amax>>23)&0xFF) - 39)<<23));
    if(!(fabsf(x)<=amax)||isnan(x)) continue;
    if (x != 0 && fabsf(x) < 0x1p-100f) continue;
    float r=1.0f/d, q=x*r, res=fmaf(-q,d,x), q1=copysignf(fmaf(res,r,q),x);
    float want=x/d; ++n;
    if(memcmp(&q1,&want,4)){ if(bad<10) printf("x=%a d=%a q1=%a want=%a\n",x,d,q1,want); ++bad; }
  }
  printf("n=%ld bad=%ld\n",n,bad);
}
