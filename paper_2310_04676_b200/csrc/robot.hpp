// Host-side robot model: the reference's versioned `.robot` descriptor format
// (parse_robot, proj/src/robot_model.cpp:191-283) and its invariants
// (validate_model, :133-161), re-written without Eigen. The parsed chain is
// packed into the device joint table (kernels.cuh: RobotTable) once per env.
#pragma once

#include <array>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace sg {

// Exception types of proj/include/scalpel/errors.hpp:23-48; the C-ABI maps
// ConfigError (and ParseError) to SG_ERR_CONFIG, SimError to SG_ERR_SIM.
class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
class ParseError : public ConfigError {
 public:
  ParseError(const std::string& origin, int line, const std::string& msg)
      : ConfigError(origin + ":" + std::to_string(line) + ": " + msg), origin_(origin), line_(line) {}
  const std::string& origin() const { return origin_; }
  int line() const { return line_; }

 private:
  std::string origin_;
  int line_;
};
class SimError : public std::runtime_error {
 public:
  explicit SimError(const std::string& m) : std::runtime_error(m) {}
};

enum class JointKind { Revolute = 0, Prismatic = 1, Fixed = 2 };

using Vec3 = std::array<double, 3>;
using Quat = std::array<double, 4>;  // w, x, y, z

struct JointSpec {  // robot_model.hpp:33-43
  std::string name;
  JointKind kind = JointKind::Revolute;
  Vec3 axis{0, 0, 1};
  Vec3 origin_translation{0, 0, 0};
  Quat origin_rotation{1, 0, 0, 0};
  double limit_lo = 0, limit_hi = 0, velocity_limit = 0, effort_limit = 0;
};

struct RobotModel {  // robot_model.hpp:47-61
  std::string name;
  int format_version = 1;
  std::vector<JointSpec> joints;
  Vec3 tip_position{0, 0, 0};
  Quat tip_orientation{1, 0, 0, 0};
  std::optional<int> jaw_joint;
  int dof_count = 0;
  std::vector<int> dof_to_joint;

  const JointSpec& dof_joint(int d) const { return joints[dof_to_joint[d]]; }
  int jaw_dof() const;                    // -1 if none
  std::vector<double> mid_configuration() const;
};

RobotModel parse_robot(std::string_view text, const std::string& origin);
RobotModel load_robot(const std::string& path);
RobotModel resolve_robot(const std::string& name_or_path);
std::vector<std::string> builtin_robot_names();

// fp64 FK on the host (used once per env for the workspace centre,
// envs.cpp:161-162). Quaternion walk with Eigen's formulas.
Vec3 forward_kinematics_position(const RobotModel& m, const std::vector<double>& q);
Quat quat_from_rpy(double roll, double pitch, double yaw);

}  // namespace sg
