#include "layout.hpp"
#include <chrono>
#include <cstdio>
using namespace rhgb;
int main(){
  double a=alpha_from_gamma(2.2); double C=radial_const_from_avg_degree(64.0,a);
  Params p(1ull<<24,a,C,7,64);
  for(int r=0;r<3;r++) make_layout(p);
  auto t0=std::chrono::steady_clock::now(); int N=50; unsigned long s=0;
  for(int r=0;r<N;r++){ auto L=make_layout(p); s+=L.counts[0];}
  auto t1=std::chrono::steady_clock::now();
  printf("layout %.3f ms (%lu)\n", std::chrono::duration<double,std::milli>(t1-t0).count()/N, s);
}
