// ORACLE probe — test infrastructure only.
// The reference builds with g++; `Eigen::Vector3d(rng.normal(..), rng.normal(..),
// rng.normal(..))` (proj/src/envs.cpp:232-234) has unspecified argument
// evaluation order in C++. This probe shows g++ evaluates constructor
// arguments right-to-left (prints "3 2 1 | 6 5 4"), so the first Box-Muller
// draw of each goal attempt lands in z. The oracle and the device follow it.
#include <cstdio>
struct V3 { double x,y,z; V3(const double& a, const double& b, const double& c): x(a),y(b),z(c) {} };
template<typename S> struct M { S d[3]; M(const S& a, const S& b, const S& c){d[0]=a;d[1]=b;d[2]=c;} };
static int ctr = 0;
__attribute__((noinline)) double draw(double mu, double s) { return mu + s * (++ctr); }
int main(){ V3 v(draw(0,1), draw(0,1), draw(0,1)); M<double> m(draw(0,1), draw(0,1), draw(0,1));
 printf("%g %g %g | %g %g %g\n", v.x, v.y, v.z, m.d[0], m.d[1], m.d[2]); }
