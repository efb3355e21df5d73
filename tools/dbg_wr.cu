#include <cstdio>
#include <cmath>
#include "dbg_vals.h"
__global__ void k(double* out) {
  double x0=X[0], x1=X[1], x2=X[2];
  double uf = rint(120.0 * x0 / x2 + 23.5);
  double vf = rint(120.0 * x1 / x2 + 23.5);
  double ox = (uf - 23.5) / 120.0 * D, oy = (vf - 23.5) / 120.0 * D;
  double dx = ox - x0, dy = oy - x1, dz = D - x2;
  out[0]=uf; out[1]=vf; out[2]=sqrt(dx*dx+dy*dy+dz*dz); out[3]=G[0]*NR[0]+G[1]*NR[1]+G[2]*NR[2];
  out[4]=G[0]*G[0]+G[1]*G[1]+G[2]*G[2];
  out[5] = 120.0 * x0 / x2 + 23.5;
}
int main(){ double* d; cudaMalloc(&d, 64); k<<<1,1>>>(d); double h[8]; cudaMemcpy(h,d,48,cudaMemcpyDeviceToHost);
 printf("uf %g vf %g dist %.17g cos %.17g gg %.17g uraw %.17g\n",h[0],h[1],h[2],h[3],h[4],h[5]); return 0;}
